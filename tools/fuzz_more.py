"""Extended randomised parity sweep (300 more seeds of tests/test_gpu_fuzz.py cases) vs the oracle; run on a GPU box."""
import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import oracle, paper_2508_00441_b200 as oz
from conftest import bits, spread_matrix
from test_gpu_fuzz import _case
bad = 0; ran = 0
for seed in range(1000, 1300):
    m, n, k, t2, t3, kb, emu, ms, order, cut, phi = _case(seed)
    rng = np.random.default_rng(seed)
    A = spread_matrix(rng, m, k, phi); B = spread_matrix(rng, k, n, phi)
    params = oz.compute_params(53, oz.get_format(t2).mant_bits, oz.get_format(t3).mant_bits, kb or k)
    if not params.feasible: continue
    try:
        Cref, info = oracle.oz_gemm(A, B, t2, t3, kb, emu, ms, order, cut)
    except ValueError:
        continue
    cfg = oz.GemmConfig(oz.get_format(t2), oz.get_format(t3), k_block=kb, fp64_emulation=emu, max_slices=ms,
                        accumulation_order=order, pair_cutoff=cut)
    res = oz.oz_gemm(A, B, cfg); ran += 1
    nb = int(np.sum(bits(res.C) != bits(Cref)))
    if nb: bad += 1; print("MISMATCH", seed, (m, n, k, t2, t3, kb, emu, ms, order, cut, phi), nb)
print("ran", ran, "bad", bad)
