"""Randomised GPU parity sweep: seeded random shapes (ragged m, n, k), formats,
accumulation types, k-blocking, max_slices, pair order, pair cutoff, emulated
accumulation and value ranges; every C must equal the CPU oracle bit for bit.
Complements the hand-picked cases in test_gpu_parity.py."""

import numpy as np
import pytest

from conftest import bits, spread_matrix

pytestmark = pytest.mark.gpu

FMTS = [("fp8e4m3", "fp32"), ("fp8e4m3", "fp16"), ("fp16", "fp32"), ("bf16", "fp32"), ("fp8e5m2", "fp32"),
        ("fp6e3m2", "fp32")]


def _case(seed):
    r = np.random.default_rng(seed)
    m, n = int(r.integers(1, 420)), int(r.integers(1, 420))
    k = int(r.integers(1, 900))
    t2, t3 = FMTS[int(r.integers(0, len(FMTS)))]
    kb = 0 if r.random() < 0.6 else int(r.integers(1, k + 1))
    emu = bool(r.random() < 0.25)
    ms = None if r.random() < 0.7 else int(r.integers(1, 8))
    order = "smallest-first" if r.random() < 0.7 else "largest-first"
    cut = None if r.random() < 0.7 else int(r.integers(0, 14))
    phi = float(r.choice([0.0, 0.5, 2.0, 5.0]))
    return m, n, k, t2, t3, kb, emu, ms, order, cut, phi


@pytest.mark.parametrize("seed", range(100))
def test_random_cases_bitwise(cuda, seed):
    import oracle
    import paper_2508_00441_b200 as oz

    m, n, k, t2, t3, kb, emu, ms, order, cut, phi = _case(seed)
    rng = np.random.default_rng(1000 + seed)
    A = spread_matrix(rng, m, k, phi)
    B = spread_matrix(rng, k, n, phi)
    if seed % 7 == 3:  # exact zeros: whole rows / columns and scattered entries
        A[rng.random(A.shape) < 0.2] = 0.0
        A[: max(1, m // 5)] = 0.0
        B[:, : max(1, n // 7)] = 0.0
    params = oz.compute_params(53, oz.get_format(t2).mant_bits, oz.get_format(t3).mant_bits, kb or k)
    if not params.feasible:
        pytest.skip("infeasible slicing parameters for this draw")
    cfg = oz.GemmConfig(oz.get_format(t2), oz.get_format(t3), k_block=kb, fp64_emulation=emu, max_slices=ms,
                        accumulation_order=order, pair_cutoff=cut)
    try:
        Cref, info = oracle.oz_gemm(A, B, t2, t3, kb, emu, ms, order, cut)
    except ValueError:
        pytest.skip("infeasible k-block for this draw")
    assert info["flags"] == 0
    res = oz.oz_gemm(A, B, cfg)
    assert [(b.k_lo, b.k_hi, b.s_x, b.s_y) for b in res.stats.blocks] == info["blocks"]
    nbad = int(np.sum(bits(res.C) != bits(Cref)))
    assert nbad == 0, f"case {(m, n, k, t2, t3, kb, emu, ms, order, cut, phi)}: {nbad} entries differ"
