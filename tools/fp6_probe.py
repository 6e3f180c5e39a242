"""Which bit position inside a byte does tcgen05 kind::f8f6f4 read an FP6 code
from (OZ_FP6_SHIFT)?  Compares the fp6e3m2 pipeline with the CPU oracle."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2508_00441_b200 as oz  # noqa: E402
from conftest import bits, spread_matrix  # noqa: E402

rng = np.random.default_rng(6)
A = spread_matrix(rng, 256, 320, 0.5)
B = spread_matrix(rng, 320, 200, 0.5)
f = oz.get_format("fp6e3m2")
params = oz.compute_params(53, f.mant_bits, 24, 320)
sa = oz.slice_matrix(A, "rows", f, params)
sb = oz.slice_matrix(B, "cols", f, params)
G = oz.lp_gemm(oz.LpMatrix(sa.coeff[0], f), oz.LpMatrix(sb.coeff[0], f), oz.get_format("fp32"))
bad_g = int(np.sum(G != sa.coeff[0] @ sb.coeff[0]))
res = oz.oz_gemm(A, B, oz.GemmConfig(f, oz.get_format("fp32")))
Cref, info = oracle.oz_gemm(A, B, "fp6e3m2", "fp32")
print("lp_gemm mismatches", bad_g, "oz_gemm mismatches", int(np.sum(bits(res.C) != bits(Cref))), info["blocks"])
E = sa.coeff[0] @ sb.coeff[0]
nz = E != 0
r = G[nz] / E[nz]
print("ratio stats", np.unique(np.round(r[:2000], 4))[:12], "G sample", G.ravel()[:4], "E sample", E.ravel()[:4])
print("coeff sample", np.unique(sa.coeff[0])[:10])
