"""A/B: pair-GEMM schedule (oz_set_pair_schedule 0 overlapped / 1 exclusive
epilogue windows), K3 device time and C hash, for several sizes and modes."""
import hashlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from paper_2508_00441_b200 import _lib  # noqa: E402
from bench import gpu_inputs  # noqa: E402

f8, f16, f32 = oz.get_format("fp8e4m3"), oz.get_format("fp16"), oz.get_format("fp32")
cases = [(1024, oz.GemmConfig(f8, f32)), (2048, oz.GemmConfig(f8, f32)), (8192, oz.GemmConfig(f8, f32)),
         (8192, oz.GemmConfig(f8, f32, pair_cutoff=11)), (8192, oz.GemmConfig(f16, f32, k_block=1024)),
         (8192, oz.GemmConfig(f8, f32, fp64_emulation=True, pair_cutoff=11))]
for n, cfg in cases:
    A, _ = gpu_inputs(torch, n, n, 8, 0.5, 1000, "cuda")
    _, B = gpu_inputs(torch, 8, n, n, 0.5, 2000, "cuda")
    C = torch.empty((n, n), dtype=torch.float64, device="cuda")
    for rnd in range(2):
        for mode in (0, 1):
            _lib.call("oz_set_pair_schedule", mode)
            oz.oz_gemm_device(A, B, cfg, out=C)
            ts = []
            for _ in range(3):
                _, st = oz.oz_gemm_device(A, B, cfg, out=C)
                ts.append(st.t_gemm * 1e3)
            h = hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()[:10]
            print(f"n={n} kb={cfg.k_block} t2={cfg.type2.name} cut={cfg.pair_cutoff} emu={cfg.fp64_emulation} "
                  f"sched={mode}: K3 {min(ts):9.3f} ms C {h}", flush=True)
    del A, B, C
_lib.call("oz_set_pair_schedule", 0)
