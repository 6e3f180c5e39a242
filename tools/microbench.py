"""Arithmetic-throughput probes (DADD vs integer-emulated add vs int64 add vs FFMA)
for choosing the fused epilogue's accumulation path.  Not part of the product."""
import ctypes
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
SO = HERE / "libmicro.so"


def build():
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "-shared", "-Xcompiler", "-fPIC", "-o", str(SO), str(HERE / "microbench.cu")], check=True)


def main(out=None):
    if not SO.exists():
        build()
    lib = ctypes.CDLL(str(SO))
    lib.micro_run.restype = ctypes.c_float
    lib.micro_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    blocks, iters = 148 * 8, 4096
    res = {}
    for kind, name in enumerate(["dadd", "emu_add", "iadd64", "ffma"]):
        ms = lib.micro_run(kind, blocks, iters)
        ops = blocks * 256 * 16 * iters
        res[name] = {"ms": ms, "Gops_per_s": ops / (ms / 1e3) / 1e9, "ops_per_clk_per_sm_at_1.9GHz":
                     ops / (ms / 1e3) / 148 / 1.9e9}
        print(name, json.dumps(res[name]))
    lib.micro_mma_rate.restype = ctypes.c_double
    lib.micro_mma_rate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    for cta, n in ((1, 128), (1, 256), (2, 128), (2, 192), (2, 256)):
        r = lib.micro_mma_rate(cta, n, 20000)
        res[f"mma_fp8_cta{cta}_n{n}"] = {"macs_per_clk_per_sm": r, "frac_of_8192": r / 8192}
        print(f"mma fp8 cta_group::{cta} N={n}: {r:.0f} MAC/clk/SM ({r / 8192:.2f} of 8192)", flush=True)
    lib.micro_side.restype = None
    lib.micro_side.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_double)]
    mr, sr = ctypes.c_double(), ctypes.c_double()
    side_iters_by = [0, 20000, 40000, 40000, 1000, 40000]
    for side, name in enumerate(["none", "dadd", "iadd64", "ffma", "fast_add_int", "imad32"]):
        si = side_iters_by[side]
        for mma_iters, side_iters in ((20000, si), (0, si)) if side else ((20000, 0),):
            lib.micro_side(side, mma_iters, side_iters, ctypes.byref(mr), ctypes.byref(sr))
            key = f"side_{name}_mma{int(mma_iters > 0)}_side{int(side_iters > 0)}"
            res[key] = {"mma_macs_per_clk_per_sm": mr.value, "side_ops_per_clk_per_sm": sr.value}
            print(f"{key}: MMA {mr.value:.0f} MAC/clk/SM, side {sr.value:.2f} op/clk/SM", flush=True)
    # Is a DADD side load blocked for the whole MMA stream?  Side work small enough
    # to finish well inside the MMA window: its duration should then be short.
    lib.micro_side_n.restype = None
    lib.micro_side_n.argtypes = lib.micro_side.argtypes
    for n in (128, 192, 256):
        for si in (250, 1000, 4000):
            lib.micro_side_n(n, 20000, si, ctypes.byref(mr), ctypes.byref(sr))
            mma_cyc = 20000 * 4 * 128 * n * 32 / mr.value if mr.value else 0
            side_cyc = 256 * 16 * si / sr.value if sr.value else 0
            key = f"window_dadd_n{n}_side{si}"
            res[key] = {"mma_cycles": mma_cyc, "side_cycles": side_cyc, "side_ops": 256 * 16 * si,
                        "side_cycles_alone_at_62.8": 256 * 16 * si / 62.8}
            print(key, json.dumps(res[key]), flush=True)
    if out:
        Path(out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
