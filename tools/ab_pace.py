"""A/B of cross-CTA pacing slack and raster band height for the pair GEMM
(scheduling only; C is bitwise unchanged): n = 8192, fixed-step cutoff 11 and
reference defaults.  Prints min device K3 time of 3 calls per setting, two rounds."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from paper_2508_00441_b200 import _lib, ozgemm  # noqa: E402
from bench import gpu_inputs  # noqa: E402

n = 8192
A, _ = gpu_inputs(torch, n, n, 8, 0.5, 1000, "cuda")
_, B = gpu_inputs(torch, 8, n, n, 0.5, 2000, "cuda")
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
f8, f32 = oz.get_format("fp8e4m3"), oz.get_format("fp32")
cfgs = {"fixed11": oz.GemmConfig(f8, f32, pair_cutoff=11, slice_exponents="fixed"), "defaults": oz.GemmConfig(f8, f32)}
for rnd in range(2):
    for name, cfg in cfgs.items():
        for slack, group in ((2, 8), (0, 8), (1, 8), (4, 8), (8, 8), (2, 4), (2, 16), (2, 32)):
            ozgemm.PACE_SLACK = slack
            _lib.set_pair_variant(0, 0, group)
            oz.oz_gemm_device(A, B, cfg, out=C)
            ts = []
            for _ in range(3 if name == "fixed11" else 2):
                _, st = oz.oz_gemm_device(A, B, cfg, out=C)
                ts.append(st.t_gemm * 1e3)
            print(f"round {rnd} {name:8s} slack {slack} group {group:2d}: K3 {min(ts):8.2f} ms", flush=True)
_lib.set_pair_variant(0, 0, 0)
