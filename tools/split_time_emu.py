"""Device time of the row split, HW vs emulated (adaptive and fixed-step).
usage: split_time_emu.py rows kb"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from paper_2508_00441_b200.slicing import split_deferred  # noqa: E402
from bench import gpu_inputs  # noqa: E402

rows, kb = int(sys.argv[1]), int(sys.argv[2])
X, _ = gpu_inputs(torch, rows, kb, 8, 0.5, 1000, "cuda")
f = oz.get_format("fp8e4m3")
params = oz.compute_params(53, f.mant_bits, 24, kb)
for occ in (2,):
    for name, emu, kw in (("hw-adaptive", False, {}), ("emu-adaptive", True, {}),
                          ("emu-fixed12", True, {"fixed": True, "max_planes": 12})):
        ts = []
        for rep in range(4):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            e[0].record()
            ds = split_deferred(X, f, params, emu, **kw)
            e[1].record()
            torch.cuda.synchronize()
            ts.append(e[0].elapsed_time(e[1]))
            del ds
        print(f"occ={occ} {name} rows={rows} kb={kb}: " + " ".join(f"{t:.2f}" for t in ts[1:]) + " ms", flush=True)
