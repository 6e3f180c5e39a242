"""Large single-GPU Ozaki DGEMM (e.g. n = 65536, panelled): device-timed
FP64-equivalent TFLOPS and max rel error of a row sample vs the DD oracle and
vs cuBLAS DGEMM.  Not part of the product; see DESIGN.md §6."""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from bench import gpu_inputs  # noqa: E402
from paper_2508_00441_b200 import _lib  # noqa: E402
from paper_2508_00441_b200.ozgemm import _panel_plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--phi", type=float, default=0.5)
ap.add_argument("--pair-cutoff", type=int, default=None)
ap.add_argument("--rows", type=int, default=64)
ap.add_argument("--out", default=None)
a = ap.parse_args()
n = a.n
A, _ = gpu_inputs(torch, n, n, 8, a.phi, 1000, "cuda")
_, B = gpu_inputs(torch, 8, n, n, a.phi, 2000, "cuda")
cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), pair_cutoff=a.pair_cutoff)
torch.cuda.empty_cache()  # release the generator's temporaries before planning panels
plan = _panel_plan(n, n, n, 1, torch)
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
C, st = oz.oz_gemm_device(A, B, cfg, out=C)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
r = a.rows
Cdd = torch.empty((r, n), dtype=torch.float64, device="cuda")
_lib.call("oz_dd_gemm", A[:r].contiguous().data_ptr(), B.data_ptr(), Cdd.data_ptr(), r, n, n, _lib.stream_ptr(torch))
Cc = torch.matmul(A[:r], B)
d, o, c = Cdd.cpu().numpy(), C[:r].cpu().numpy(), Cc.cpu().numpy()
nz = d != 0
rel = lambda X: float(np.max(np.abs(X[nz] - d[nz]) / np.abs(d[nz])))  # noqa: E731
res = {"n": n, "phi": a.phi, "pair_cutoff": a.pair_cutoff, "panels": plan, "ms": ms,
       "tflops_fp64_equiv": 2.0 * n ** 3 / (ms / 1e3) / 1e12, "t_slice_s": st.t_slice, "t_gemm_s": st.t_gemm,
       "s": [(b.s_x, b.s_y) for b in st.blocks], "gemm_count": st.gemm_count,
       "max_rel_err_ozaki": rel(o), "max_rel_err_cublas_dgemm": rel(c), "rows_checked": r,
       "wall_s": time.perf_counter() - t0}
print(json.dumps(res))
if a.out:
    Path(a.out).write_text(json.dumps(res, indent=1))
