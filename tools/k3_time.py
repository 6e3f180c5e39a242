"""K3 device time (min of 3 calls) at n = 8192 for defaults and pair_cutoff 11,
and a hash of C (bitwise comparison across library builds).  Diagnostics."""
import hashlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from bench import gpu_inputs  # noqa: E402

n = 8192
A, _ = gpu_inputs(torch, n, n, 8, 0.5, 1000, "cuda")
_, B = gpu_inputs(torch, 8, n, n, 0.5, 2000, "cuda")
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for cut in (None, 11):
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), pair_cutoff=cut)
    oz.oz_gemm_device(A, B, cfg, out=C)
    ts = []
    for _ in range(3):
        _, st = oz.oz_gemm_device(A, B, cfg, out=C)
        ts.append(st.t_gemm * 1e3)
    h = hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"{tag} cut={cut}: K3 min {min(ts):7.2f} ms runs {[round(t, 1) for t in ts]} C {h}", flush=True)
