"""FP6 (fp6e3m2) through the fused pipeline vs the CPU oracle: packed 6-bit
slice planes, TMA 16U6_ALIGN16B unpacking, kind::f8f6f4 E3M2 MMAs."""
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
for m, n, k in ((256, 200, 320), (130, 64, 100), (512, 384, 1024)):
    A = spread_matrix(rng, m, k, 0.5)
    B = spread_matrix(rng, k, n, 0.5)
    f = oz.get_format("fp6e3m2")
    res = oz.oz_gemm(A, B, oz.GemmConfig(f, oz.get_format("fp32")))
    Cref, info = oracle.oz_gemm(A, B, "fp6e3m2", "fp32")
    d = bits(res.C) != bits(Cref)
    print((m, n, k), "mismatches", int(d.sum()), "of", m * n, info["blocks"],
          "max rel diff", float(np.max(np.abs(res.C - Cref) / np.maximum(np.abs(Cref), 1e-300))))
