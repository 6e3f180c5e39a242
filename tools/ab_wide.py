"""A/B: CTA-pair tile 256 x 192 vs 256 x 256 for the fixed-step grouped mode
(n = 8192, cutoff 11), alternating in one process; K3 device time and C hash."""
import hashlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from paper_2508_00441_b200 import _lib  # noqa: E402
from bench import gpu_inputs  # noqa: E402

n = 8192
A, _ = gpu_inputs(torch, n, n, 8, 0.5, 1000, "cuda")
_, B = gpu_inputs(torch, 8, n, n, 0.5, 2000, "cuda")
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), pair_cutoff=11, slice_exponents="fixed")
for rnd in range(4):
    for tn in (192, 256):
        _lib.set_pair_variant(2, tn, 0)
        oz.oz_gemm_device(A, B, cfg, out=C)
        ts = []
        for _ in range(3):
            _, st = oz.oz_gemm_device(A, B, cfg, out=C)
            ts.append(st.t_gemm * 1e3)
        h = hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()[:10]
        print(f"round {rnd} N={tn}: K3 min {min(ts):7.2f} ms runs {[round(t, 2) for t in ts]} C {h}", flush=True)
_lib.set_pair_variant(0, 0, 0)
