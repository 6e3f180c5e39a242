"""Per-pair timeline of K3 for unit 0 (OZ_TRACE): MMA warp wait on a free
accumulator, MMA issue span, epilogue wait for a full accumulator and its
processing time, in SM cycles.  Diagnostics only."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from bench import gpu_inputs  # noqa: E402

cut = int(sys.argv[1]) if len(sys.argv) > 1 else 11
n = 8192
A, _ = gpu_inputs(torch, n, n, 8, 0.5, 1000, "cuda")
_, B = gpu_inputs(torch, 8, n, n, 0.5, 2000, "cuda")
cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), pair_cutoff=cut)
oz.oz_gemm_device(A, B, cfg)
cap = 4096
tr = torch.zeros(cap * 8, dtype=torch.int64, device="cuda")
os.environ["OZ_TRACE"] = f"{tr.data_ptr():x}:{cap}"
oz.oz_gemm_device(A, B, cfg)
torch.cuda.synchronize()
del os.environ["OZ_TRACE"]
t = tr.cpu().numpy().reshape(cap, 8).astype(np.float64)
t = t[t[:, 2] > 0]
mma_wait = t[:, 1] - t[:, 0]
mma_span = t[1:, 0] - t[:-1, 0]
epi_wait = t[:, 4] - t[:, 3]
epi_proc = t[:, 5] - t[:, 4]
full_wait = t[:, 6]
epi_reg = t[:, 7] - t[:, 4]
epi_tm = t[:, 5] - t[:, 7]
print(f"pairs traced {len(t)}")
for name, v in (("mma wait acc_empty", mma_wait), ("mma pair period", mma_span), ("epi wait acc_full", epi_wait),
                ("epi processing", epi_proc), ("mma full waits/pair", full_wait), ("epi register part", epi_reg),
                ("epi TMEM part", epi_tm)):
    print(f"{name:20s} mean {v.mean():9.0f}  p50 {np.median(v):9.0f}  p90 {np.percentile(v, 90):9.0f}  "
          f"max {v.max():9.0f} cycles")
print("mma wait share of period", mma_wait[1:].sum() / mma_span.sum())
# first pairs of each tile (where the waits cluster?)
per = cut + 1
print("epi processing by pair index mod tile (first 4):", [float(np.mean(epi_proc[i::78])) for i in range(4)])
