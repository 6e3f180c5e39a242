"""Bitwise parity at the BASELINE sizes, on the multi-wave persistent path that
produces the benchmark numbers.

* Config 1 in full (n = m = k = 1024, phi = 0.5, fp8e4m3/fp32, reference
  defaults): the GPU's C has the same sha256 as the C the REFERENCE computed
  (tests/golden/config1.json, made by gen_big_golden.py running ozdgemm).
* n = 4096 and 8192 (5-19 waves of 256 x 192 tiles over 74 CTA pairs): sampled
  C blocks — rows and columns spread over every raster band and several tile
  waves — against the CPU oracle run on just those A rows and B columns.  Slicing
  is row/column-local and the pairs a sample lacks (its s may be below the
  global s) only add +0 terms, so the sample's oracle C is exactly the full C's
  block.  Options: reference defaults, emulated FP64, FP16 slices with
  k_block = 1024, pair_cutoff = 11, and phi = 4.
* Run-to-run determinism of the full n = 4096 C.
"""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).view(np.uint64).tobytes()).hexdigest()


def test_config1_full_matches_reference(cuda):
    import paper_2508_00441_b200 as oz

    g = json.loads((GOLD / "config1.json").read_text())
    n, phi = g["n"], g["phi"]
    rng = np.random.default_rng(g["seed"])
    A = (rng.random((n, n)) - 0.5) * np.exp(phi * rng.standard_normal((n, n)))
    B = (rng.random((n, n)) - 0.5) * np.exp(phi * rng.standard_normal((n, n)))
    assert sha(A) == g["sha256_A"] and sha(B) == g["sha256_B"], "numpy stream differs from the generator's"
    res = oz.oz_gemm(A, B, oz.GemmConfig(oz.get_format(g["type2"]), oz.get_format(g["type3"])))
    assert [[b.k_lo, b.k_hi, b.s_x, b.s_y] for b in res.stats.blocks] == g["blocks"]
    assert res.stats.gemm_count == g["gemm_count"]
    for i, j, v in g["samples"]:
        assert int(res.C.view(np.uint64)[i, j]) == v
    assert sha(res.C) == g["sha256_C"]


def sample_index(n, groups=6, width=32):
    """`groups` runs of `width` consecutive indices spread from the first to the
    last tile (different raster bands / tile waves), always including the end."""
    starts = np.linspace(0, n - width, groups).astype(int)
    starts = (starts // 8) * 8
    starts[-1] = n - width
    return np.unique(np.concatenate([np.arange(s, s + width) for s in starts]))


def device_inputs(torch, n, phi, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = (torch.rand((n, n), generator=g, device="cuda", dtype=torch.float64) - 0.5) * torch.exp(
        phi * torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64))
    B = (torch.rand((n, n), generator=g, device="cuda", dtype=torch.float64) - 0.5) * torch.exp(
        phi * torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64))
    return A, B


SCALE_CASES = [
    # n, phi, type2, k_block, emu, pair_cutoff
    (8192, 0.5, "fp8e4m3", 0, False, None),
    (8192, 0.5, "fp8e4m3", 0, True, None),
    (8192, 0.5, "fp8e4m3", 0, False, 11),
    (8192, 4.0, "fp8e4m3", 0, False, None),
    (4096, 0.5, "fp8e4m3", 0, False, None),
    (4096, 0.5, "fp16", 1024, False, None),
    (4096, 4.0, "fp16", 1024, True, None),
]


@pytest.mark.parametrize("case", SCALE_CASES, ids=[f"n{c[0]}-phi{c[1]}-{c[2]}-kb{c[3]}-emu{int(c[4])}-cut{c[5]}"
                                                   for c in SCALE_CASES])
def test_sampled_blocks_bitwise_multiwave(cuda, case):
    torch = cuda
    import oracle
    import paper_2508_00441_b200 as oz

    n, phi, t2, kbk, emu, cut = case
    A, B = device_inputs(torch, n, phi, 1000 + n + int(10 * phi))
    cfg = oz.GemmConfig(oz.get_format(t2), oz.get_format("fp32"), k_block=kbk, fp64_emulation=emu,
                        pair_cutoff=cut)
    C, st = oz.oz_gemm_device(A, B, cfg)
    rows, cols = sample_index(n), sample_index(n)
    Cs = C[rows][:, cols].cpu().numpy()
    As = A[rows].cpu().numpy()
    Bs = B[:, cols].cpu().numpy()
    Cref, info = oracle.oz_gemm(As, Bs, t2, "fp32", kbk, emu, None, "smallest-first", cut)
    assert info["flags"] == 0
    # the sample's slice counts never exceed the full problem's
    for (lo, hi, sx, sy), b in zip(info["blocks"], st.blocks):
        assert (lo, hi) == (b.k_lo, b.k_hi) and sx <= b.s_x and sy <= b.s_y
    nbad = int(np.sum(Cs.view(np.uint64) != Cref.view(np.uint64)))
    assert nbad == 0, f"{nbad} of {Cs.size} sampled entries differ"


@pytest.mark.parametrize("cut,emu", [(11, False), (10, True), (None, False)])
def test_fixed_step_sampled_blocks_n8192(cuda, cut, emu):
    """The opt-in fast mode (fixed-step slices, level-grouped accumulation) at the
    headline size: sampled C blocks over all tile waves, bitwise against the CPU
    restatement on the same A rows / B columns."""
    torch = cuda
    import oracle
    import paper_2508_00441_b200 as oz

    n = 8192
    A, B = device_inputs(torch, n, 0.5, 4242)
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), fp64_emulation=emu, pair_cutoff=cut,
                        slice_exponents="fixed")
    C, st = oz.oz_gemm_device(A, B, cfg)
    rows, cols = sample_index(n), sample_index(n)
    Cs = C[rows][:, cols].cpu().numpy()
    # pad the sample's slices to the full problem's counts: pair groups then match
    Cref, blocks = oracle.oz_gemm_fixed(A[rows].cpu().numpy(), B[:, cols].cpu().numpy(), "fp8e4m3", "fp32", 0,
                                        None, "smallest-first", cut,
                                        pad_to=[(st.blocks[0].s_x, st.blocks[0].s_y)])
    assert (blocks[0][2], blocks[0][3]) == (st.blocks[0].s_x, st.blocks[0].s_y)
    nbad = int(np.sum(Cs.view(np.uint64) != Cref.view(np.uint64)))
    assert nbad == 0, f"{nbad} of {Cs.size} sampled entries differ"


def test_full_c_deterministic(cuda):
    torch = cuda
    import paper_2508_00441_b200 as oz

    A, B = device_inputs(torch, 4096, 0.5, 77)
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"))
    C1, _ = oz.oz_gemm_device(A, B, cfg)
    h1 = hashlib.sha256(C1.view(torch.int64).cpu().numpy().tobytes()).hexdigest()
    for _ in range(2):
        C2, _ = oz.oz_gemm_device(A, B, cfg)
        assert hashlib.sha256(C2.view(torch.int64).cpu().numpy().tobytes()).hexdigest() == h1
