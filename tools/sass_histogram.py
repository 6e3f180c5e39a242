"""Per-kernel SASS opcode histogram of liboz_b200.so (cuobjdump -sass).

    python tools/sass_histogram.py [lib] > profiles/sass_opcodes_r02.txt

For each kernel: tensor-core MMAs (UTC*MMA), TMEM loads/stores (LDTM/STTM), TMA
loads (UTMALDG), FP64 instructions (D*, F2F.F64, I2F.F64, ...), and the total
instruction count.  The emulated-FP64 path (pair_gemm_kernel<true, ...>, the
split_fused_kernel<..., true> instantiations and their helper kernels) must show
0 FP64 instructions (north_star; enforced by tests/test_capi.py).
"""

from __future__ import annotations

import re
import shutil
import subprocess
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
FP64 = re.compile(r"^(DFMA|DADD|DMUL|DSETP|DMNMX|DSET|DRCP|DMMA|F2F\.F64|F2F\.F32\.F64|I2F\.F64|F2I\.F64)")
CLASSES = {
    "UTC*MMA": re.compile(r"^UTC\w*MMA"),
    "LDTM": re.compile(r"^LDTM"),
    "STTM": re.compile(r"^STTM"),
    "UTMALDG": re.compile(r"^UTMALDG"),
    "FP64": FP64,
}


def demangle(names):
    cf = shutil.which("c++filt")
    if not cf:
        return {n: n for n in names}
    out = subprocess.run([cf], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def histogram(lib: Path):
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([exe, "-sass", str(lib)], check=True, capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m:
            funcs[cur][m.group(1)] += 1
    return funcs


def main():
    lib = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "paper_2508_00441_b200" / "liboz_b200.so"
    funcs = histogram(lib)
    names = demangle(sorted(funcs))
    print(f"# SASS opcode histogram of {lib.name} (cuobjdump -sass); columns: " + ", ".join(CLASSES) + ", total")
    print("# FP64 = DFMA/DADD/DMUL/DSETP/DMNMX/DSET/DRCP/DMMA/F2F.F64/I2F.F64/F2I.F64")
    for raw in sorted(funcs, key=lambda k: names[k]):
        c = funcs[raw]
        row = {k: sum(v for op, v in c.items() if rx.search(op)) for k, rx in CLASSES.items()}
        fp64_ops = sorted(op for op in c if FP64.search(op))
        print(f"{names[raw]}\n    " + "  ".join(f"{k}={v}" for k, v in row.items())
              + f"  total={sum(c.values())}" + (f"  fp64_ops={fp64_ops}" if fp64_ops else ""))


if __name__ == "__main__":
    main()
