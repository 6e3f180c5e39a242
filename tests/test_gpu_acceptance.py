"""The reference's acceptance criteria (SPEC.md:468-478,
pkg/tests/test_acceptance.py:68-250) restated against the CUDA backend, at the
reference's sizes.  Criterion 1 (GEMM-count table), 4 (scalar FP64 emulation vs
hardware) and 8 (blocked counts) are host-side and live in test_host.py /
test_cli.py.

Checkers: bitwise reconstruction (2), exact float64 products of the slice
planes (3, exact because every partial sum is a small multiple of the slice
grid), the GPU's own hardware-FP64 path (5), and for 6/7 the CPU double-double
oracle, which tests/test_oracle_golden.py pins bit for bit to the reference's
exact ref_gemm on these very inputs.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _decode_table(torch, fmt):
    from paper_2508_00441_b200.formats import decode_codes

    if fmt.name in ("fp16", "bf16"):
        return None
    t = decode_codes(np.arange(256, dtype=np.uint8), fmt.name)
    return torch.from_numpy(np.nan_to_num(t)).cuda()


def _pow2(torch, e):
    """2^e as float64, assembled from bits (exact for normal e)."""
    return ((e.long() + 1023) << 52).view(torch.float64)


def _plane_values(torch, ds, p, table):
    codes = ds.planes[p].view(torch.uint8)[:, : ds.kb] if table is not None else None
    if table is not None:
        return table[codes.long()]
    h = ds.planes[p].view(torch.int16)[:, : ds.kb]
    if ds.fmt.name == "fp16":
        return h.view(torch.float16).double()
    return (h.int() << 16).view(torch.float32).double()


@pytest.mark.parametrize("fmt_name", ["fp16", "fp8e4m3"])
@pytest.mark.parametrize("k", [8, 1024, 16384])
@pytest.mark.parametrize("dist", ["uniform", "spread"])
def test_criterion_2_reconstruction_exact(cuda, fmt_name, k, dist):
    """10^4 vectors per (format, k, distribution): sum_p ldexp(coeff_p, e_p)
    reproduces every input bit for bit (test_acceptance.py:68-95)."""
    torch = cuda
    import paper_2508_00441_b200 as oz
    from paper_2508_00441_b200.slicing import split_rows_device

    fmt = oz.get_format(fmt_name)
    params = oz.compute_params(53, fmt.mant_bits, 24, k)
    table = _decode_table(torch, fmt)
    g = torch.Generator(device="cuda").manual_seed(2024 + k)
    n_vec, done, fails = 10_000, 0, 0
    chunk = min(n_vec, max(1, 40_000_000 // k))
    while done < n_vec:
        rows = min(chunk, n_vec - done)
        X = 1.0 + 9.0 * torch.rand((rows, k), generator=g, device="cuda", dtype=torch.float64)
        if dist == "spread":
            X = X * _pow2(torch, torch.randint(-20, 21, (rows, k), generator=g, device="cuda"))
        ds, _ = split_rows_device(X, fmt, params, False)
        rec = torch.zeros_like(X)
        for p in range(ds.s):
            rec += _plane_values(torch, ds, p, table) * _pow2(torch, ds.expo[p])[:, None]
        fails += int((rec.view(torch.int64) != X.view(torch.int64)).any(dim=1).sum())
        done += rows
    assert fails == 0, f"{fails} of {n_vec} vectors not reconstructed bit for bit"


FEASIBLE = [(t2, t3, k) for k in (8, 256, 4096)
            for t2 in ("fp16", "bf16", "fp8e4m3", "fp8e5m2", "fp6e3m2", "fp6e2m3")
            for t3 in ("fp32", "fp16")]


@pytest.mark.parametrize("t2,t3,k", FEASIBLE)
def test_criterion_3_error_free_pair_gemms(cuda, t2, t3, k):
    """Every feasible (type2, type3) at k = 8 / 256 / 4096, 100 x 100 instances,
    pairs (p, q) in {0, s/2, s-1}^2: lp_gemm on the tensor cores equals the exact
    product (test_acceptance.py:100-136).  fp6e2m3 is SlicingInfeasible wherever
    its subnormal range cannot hold the slice quantum (the only allowed skip)."""
    import paper_2508_00441_b200 as oz

    f2, f3 = oz.get_format(t2), oz.get_format(t3)
    params = oz.compute_params(53, f2.mant_bits, f3.mant_bits, k)
    if not params.feasible:
        pytest.skip("infeasible combination (no GEMM count in the table)")
    rng = np.random.default_rng(3 + k)
    A = 1.0 + 9.0 * rng.random((100, k))
    B = 1.0 + 9.0 * rng.random((k, 100))
    try:
        sa = oz.slice_matrix(A, "rows", f2, params)
        sb = oz.slice_matrix(B, "cols", f2, params)
    except oz.SlicingInfeasible:
        assert t2 == "fp6e2m3"
        import oracle

        # the reference's representability rule: some coefficient needs a finer quantum than E2M3 holds
        coeff, _, _, _ = oracle.slice_matrix(A, "rows", params.rho)
        assert any(np.any(np.abs(c[c != 0]) < 2.0 ** -3) or np.any((c * 8) % 1 != 0) for c in coeff)
        return
    for p in sorted({0, sa.s // 2, sa.s - 1}):
        for q in sorted({0, sb.s // 2, sb.s - 1}):
            G = oz.lp_gemm(oz.LpMatrix(sa.coeff[p], f2, _validated=True),
                           oz.LpMatrix(sb.coeff[q], f2, _validated=True), f3)
            exact = sa.coeff[p] @ sb.coeff[q]  # exact: partial sums are small grid multiples
            assert np.array_equal(G, exact), (p, q)


@pytest.mark.parametrize("n", [16, 64, 256])
@pytest.mark.parametrize("fmt_name", ["fp16", "fp8e4m3"])
def test_criterion_5_emulation_bitwise_end_to_end(cuda, n, fmt_name):
    """oz_gemm with integer-emulated accumulation == hardware FP64, bit for bit
    (test_acceptance.py:166-183), and both == the CPU oracle."""
    import oracle
    import paper_2508_00441_b200 as oz

    rng = np.random.default_rng(5 + n)
    A = 1.0 + 9.0 * rng.random((n, n))
    B = 1.0 + 9.0 * rng.random((n, n))
    f, f32 = oz.get_format(fmt_name), oz.get_format("fp32")
    hw = oz.oz_gemm(A, B, oz.GemmConfig(f, f32)).C
    emu = oz.oz_gemm(A, B, oz.GemmConfig(f, f32, fp64_emulation=True)).C
    ref, _ = oracle.oz_gemm(A, B, fmt_name, "fp32")
    assert np.array_equal(hw.view(np.uint64), emu.view(np.uint64))
    assert np.array_equal(hw.view(np.uint64), ref.view(np.uint64))


def _rel(C, R):
    return float(np.max(np.abs(C - R) / np.abs(R)))


@pytest.fixture(scope="module")
def ref_cache():
    import oracle

    cache = {}

    def get(n, seed):
        if (n, seed) not in cache:
            rng = np.random.default_rng(seed)
            A = 1.0 + 9.0 * rng.random((n, n))
            B = 1.0 + 9.0 * rng.random((n, n))
            Cref = oracle.dd_gemm(A, B)
            cache[(n, seed)] = (A, B, Cref, _rel(oracle.naive_gemm(A, B), Cref))
        return cache[(n, seed)]

    return get


@pytest.mark.parametrize("n", [64, 256, 512])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_criterion_6_accuracy_dominance(cuda, ref_cache, n, seed):
    """max_rel_error(oz) <= max_rel_error(naive FP64) for FP16 and E4M3 slices
    (test_acceptance.py:219-233)."""
    import paper_2508_00441_b200 as oz

    A, B, Cref, err_naive = ref_cache(n, seed)
    for fmt in ("fp16", "fp8e4m3"):
        C = oz.oz_gemm(A, B, oz.GemmConfig(oz.get_format(fmt), oz.get_format("fp32"))).C
        assert _rel(C, Cref) <= err_naive, fmt


def test_criterion_7_blocked_accuracy(cuda, ref_cache):
    """FP16 slices with k_block 64 / 256 at 256^3: error within 4x naive
    (test_acceptance.py:236-248)."""
    import paper_2508_00441_b200 as oz

    A, B, Cref, err_naive = ref_cache(256, 1)
    for kb in (64, 256):
        C = oz.oz_gemm(A, B, oz.GemmConfig(oz.get_format("fp16"), oz.get_format("fp32"), k_block=kb)).C
        assert _rel(C, Cref) <= 4 * err_naive, kb
