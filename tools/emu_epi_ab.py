"""A/B of an alternative build of the library (argv[1]: .so path or 'head') for the
emulated-FP64 pair GEMM: bitwise check against the oracle, then device time of
emulated reference-default steps at n = 8192.  usage: emu_epi_ab.py head|path"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_00441_b200._lib as L  # noqa: E402

if sys.argv[1] != "head":
    L._lib = L.load(sys.argv[1])
import oracle  # noqa: E402
import paper_2508_00441_b200 as oz  # noqa: E402
from bench import gpu_inputs, _time_steps  # noqa: E402
from conftest import spread_matrix  # noqa: E402

f8, f32 = oz.get_format("fp8e4m3"), oz.get_format("fp32")
rng = np.random.default_rng(3)
A = spread_matrix(rng, 300, 1000, 1.0)
B = spread_matrix(rng, 1000, 260, 1.0)
L.set_pair_variant(1, 128, 0)
C = oz.oz_gemm(A, B, oz.GemmConfig(f8, f32, fp64_emulation=True)).C
L.set_pair_variant(0, 0, 0)
Cref, _ = oracle.oz_gemm(A, B, "fp8e4m3", "fp32", 0, True)
print(sys.argv[1], "bitwise:", np.array_equal(C.view(np.uint64), Cref.view(np.uint64)), flush=True)
n = 8192
Ad, Bd = gpu_inputs(torch, n, n, n, 0.5, 1, "cuda")
for rep in range(2):
    ms, st = _time_steps(torch, oz, Ad, Bd, oz.GemmConfig(f8, f32, fp64_emulation=True), 3)
    print(f"{sys.argv[1]} emu defaults: {ms:.2f} ms/step ({2 * n ** 3 / ms / 1e9:.2f} TF/s), K3 {st.t_gemm * 1e3:.2f} ms",
          flush=True)
