"""Dump the raw K3 per-accumulator timeline of unit 0 (OZ_TRACE; needs a
-DOZ_DIAGNOSTICS=1 build) to gpurun_out/ for offline analysis.  Diagnostics only.
usage: k3_trace_dump.py <pair_cutoff|-1> <fixed 0/1> <out.npy>"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from bench import gpu_inputs  # noqa: E402

cut = int(sys.argv[1])
fixed = bool(int(sys.argv[2]))
out = sys.argv[3]
n = 8192
A, _ = gpu_inputs(torch, n, n, 8, 0.5, 1000, "cuda")
_, B = gpu_inputs(torch, 8, n, n, 0.5, 2000, "cuda")
cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), pair_cutoff=None if cut < 0 else cut,
                    slice_exponents="fixed" if fixed else "adaptive")
oz.oz_gemm_device(A, B, cfg)
cap = 8192
tr = torch.zeros(cap * 8, dtype=torch.int64, device="cuda")
os.environ["OZ_TRACE"] = f"{tr.data_ptr():x}:{cap}"
_, st = oz.oz_gemm_device(A, B, cfg)
torch.cuda.synchronize()
del os.environ["OZ_TRACE"]
np.save(out, tr.cpu().numpy().reshape(cap, 8))
print("saved", out, "t_gemm", st.t_gemm)
