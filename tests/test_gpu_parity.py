"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
bit for bit — slices, exponents, per-row counts, s, and the final C."""

import numpy as np
import pytest

from conftest import bits, spread_matrix

pytestmark = pytest.mark.gpu


def _oz():
    import paper_2508_00441_b200 as oz

    return oz


@pytest.mark.parametrize("fmt", ["fp8e4m3", "fp16", "bf16", "fp8e5m2"])
@pytest.mark.parametrize("emu", [False, True])
@pytest.mark.parametrize("shape,phi", [((7, 33), 0.5), ((64, 1000), 4.0), ((130, 4096), 1.0)])
def test_split_rows_bitwise(cuda, fmt, emu, shape, phi):
    import oracle

    oz = _oz()
    rng = np.random.default_rng(hash((fmt, emu, shape)) % 2**32)
    X = spread_matrix(rng, *shape, phi)
    kb = shape[1]
    params = oz.compute_params(53, oz.get_format(fmt).mant_bits, 24, kb)
    ss = oz.slice_matrix(X, "rows", oz.get_format(fmt), params, "emu" if emu else "fp64")
    coeff, expo, _, s, flags = oracle.split_rows(X, params.rho, emu)
    assert flags == 0
    assert ss.s == s
    for p in range(s):
        assert np.array_equal(bits(ss.coeff[p]), bits(coeff[p])), f"coeff plane {p}"
        assert np.array_equal(ss.expo[p], expo[p].astype(np.int64)), f"expo plane {p}"


def test_split_cols_bitwise(cuda):
    import oracle

    oz = _oz()
    rng = np.random.default_rng(5)
    M = spread_matrix(rng, 300, 77, 2.0)
    params = oz.compute_params(53, 4, 24, 300)
    ss = oz.slice_matrix(M, "cols", oz.get_format("fp8e4m3"), params)
    coeff, expo, s, flags = oracle.slice_matrix(M, "cols", params.rho)
    assert ss.s == s
    for p in range(s):
        assert np.array_equal(bits(ss.coeff[p]), bits(coeff[p]))
        assert np.array_equal(ss.expo[p], expo[p])


CASES = [
    # m, n, k, phi, type2, type3, k_block, emu, max_slices, order, cutoff
    (128, 128, 128, 0.5, "fp8e4m3", "fp32", 0, False, None, "smallest-first", None),
    (192, 160, 320, 0.5, "fp8e4m3", "fp32", 0, False, None, "smallest-first", None),
    (100, 77, 333, 4.0, "fp8e4m3", "fp32", 0, False, None, "smallest-first", None),
    (256, 256, 1024, 0.5, "fp8e4m3", "fp32", 0, True, None, "smallest-first", None),
    (200, 136, 640, 1.0, "fp8e4m3", "fp32", 256, False, None, "smallest-first", None),
    (129, 257, 200, 2.0, "fp8e4m3", "fp32", 0, False, 5, "largest-first", None),
    (256, 128, 512, 0.5, "fp16", "fp32", 0, False, None, "smallest-first", None),
    (160, 96, 700, 4.0, "fp16", "fp32", 300, True, None, "smallest-first", None),
    (128, 128, 256, 0.5, "fp8e4m3", "fp16", 0, False, None, "smallest-first", None),
    (128, 200, 512, 0.5, "fp8e4m3", "fp32", 0, False, None, "smallest-first", 12),
    (64, 64, 96, 1.0, "bf16", "fp32", 0, False, None, "smallest-first", None),
    (64, 64, 96, 1.0, "fp8e5m2", "fp32", 0, False, None, "largest-first", None),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}x{c[2]}-{c[4]}-{c[5]}-kb{c[6]}-emu{int(c[7])}"
                                             f"-ms{c[8]}-{c[9][:5]}-cut{c[10]}" for c in CASES])
@pytest.mark.parametrize("skip", [True, False])
@pytest.mark.parametrize("variant", [("1", "64"), ("1", "128"), ("2", "128"), ("2", "192")],
                         ids=lambda v: f"cta{v[0]}-n{v[1]}")
def test_oz_gemm_bitwise(cuda, case, skip, variant, pair_variant):
    import oracle

    pair_variant(int(variant[0]), int(variant[1]))  # kernel variant of oz_pair_gemm

    oz = _oz()
    m, n, k, phi, t2, t3, kbk, emu, ms, order, cut = case
    rng = np.random.default_rng(m * 7 + n * 13 + k)
    A = spread_matrix(rng, m, k, phi)
    B = spread_matrix(rng, k, n, phi)
    cfg = oz.GemmConfig(oz.get_format(t2), oz.get_format(t3), k_block=kbk, fp64_emulation=emu,
                        max_slices=ms, accumulation_order=order, pair_cutoff=cut, skip_zero_pairs=skip)
    res = oz.oz_gemm(A, B, cfg)
    Cref, info = oracle.oz_gemm(A, B, t2, t3, kbk, emu, ms, order, cut)
    assert info["flags"] == 0
    assert [(b.k_lo, b.k_hi, b.s_x, b.s_y) for b in res.stats.blocks] == info["blocks"]
    nbad = int(np.sum(bits(res.C) != bits(Cref)))
    assert nbad == 0, f"{nbad}/{m * n} entries differ"


def test_device_tensors_roundtrip(cuda):
    torch = cuda
    oz = _oz()
    rng = np.random.default_rng(3)
    A = spread_matrix(rng, 256, 512, 0.5)
    B = spread_matrix(rng, 512, 128, 0.5)
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"))
    r1 = oz.oz_gemm(A, B, cfg)
    r2 = oz.oz_gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), cfg)
    assert isinstance(r2.C, torch.Tensor) and r2.C.is_cuda
    assert np.array_equal(bits(r1.C), bits(r2.C.cpu().numpy()))
    # host (pinned) torch tensors in -> host tensor out
    r3 = oz.oz_gemm(torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory(), cfg)
    assert isinstance(r3.C, torch.Tensor) and not r3.C.is_cuda and r3.C.is_pinned()
    assert np.array_equal(bits(r1.C), bits(r3.C.numpy()))


def test_lp_gemm_exact_on_slices(cuda):
    oz = _oz()
    rng = np.random.default_rng(11)
    A = spread_matrix(rng, 130, 256, 0.5)
    B = spread_matrix(rng, 256, 70, 0.5)
    f = oz.get_format("fp8e4m3")
    params = oz.compute_params(53, 4, 24, 256)
    sa = oz.slice_matrix(A, "rows", f, params)
    sb = oz.slice_matrix(B, "cols", f, params)
    for p in (0, sa.s - 1):
        for q in (0, sb.s - 1):
            G = oz.lp_gemm(oz.LpMatrix(sa.coeff[p], f), oz.LpMatrix(sb.coeff[q], f), oz.get_format("fp32"))
            assert np.array_equal(G, sa.coeff[p] @ sb.coeff[q])


@pytest.mark.parametrize("shape,fmt,emu", [((5, 20000), "fp8e4m3", False), ((3, 40000), "fp16", False),
                                           ((2, 65536), "fp8e4m3", False), ((2, 17000), "fp8e4m3", True)])
def test_split_long_rows_cluster(cuda, shape, fmt, emu):
    """kb > 16384: a cluster of CTAs shares each row (DSMEM max per slice)."""
    import oracle

    oz = _oz()
    rng = np.random.default_rng(shape[1])
    X = spread_matrix(rng, *shape, 1.0)
    params = oz.compute_params(53, oz.get_format(fmt).mant_bits, 24, shape[1])
    ss = oz.slice_matrix(X, "rows", oz.get_format(fmt), params, "emu" if emu else "fp64")
    coeff, expo, _, s, flags = oracle.split_rows(X, params.rho, emu)
    assert flags == 0 and ss.s == s
    for p in range(s):
        assert np.array_equal(bits(ss.coeff[p]), bits(coeff[p])), f"coeff plane {p}"
        assert np.array_equal(ss.expo[p], expo[p].astype(np.int64)), f"expo plane {p}"


@pytest.mark.parametrize("emu", [False, True])
def test_split_plane_cap_fallback(cuda, emu, monkeypatch):
    """Rows needing more planes than the one-pass buffer holds re-run the exact
    two-pass split; the result is unchanged."""
    import oracle
    from paper_2508_00441_b200 import slicing

    oz = _oz()
    monkeypatch.setattr(slicing, "PLANE_CAP", 3)
    monkeypatch.setattr(slicing, "PLANE_BUDGET_BYTES", 1)
    rng = np.random.default_rng(77)
    X = spread_matrix(rng, 40, 300, 4.0)
    params = oz.compute_params(53, 4, 24, 300)
    ss = oz.slice_matrix(X, "rows", oz.get_format("fp8e4m3"), params, "emu" if emu else "fp64")
    coeff, expo, _, s, flags = oracle.split_rows(X, params.rho, emu)
    assert s > 3 and ss.s == s
    for p in range(s):
        assert np.array_equal(bits(ss.coeff[p]), bits(coeff[p]))
        assert np.array_equal(ss.expo[p], expo[p].astype(np.int64))


def test_oz_gemm_long_k_bitwise(cuda):
    """k = 20000 > 16384 (cluster split) through the fused pair GEMM."""
    import oracle

    oz = _oz()
    rng = np.random.default_rng(20000)
    A = spread_matrix(rng, 40, 20000, 0.5)
    B = spread_matrix(rng, 20000, 24, 0.5)
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"))
    res = oz.oz_gemm(A, B, cfg)
    Cref, info = oracle.oz_gemm(A, B, "fp8e4m3", "fp32")
    assert info["flags"] == 0
    assert np.array_equal(bits(res.C), bits(Cref))


@pytest.mark.parametrize("case", [(300, 260, 400, 0.5, 0, None), (257, 129, 700, 4.0, 300, None),
                                  (256, 384, 512, 1.0, 0, 11)])
def test_oz_gemm_panels_bitwise(cuda, case, monkeypatch):
    """C produced panel by panel (the memory-limited path, e.g. n = 65536 on one
    GPU) is bitwise the unpanelled / oracle result, including panels whose s is
    below the global s."""
    import oracle

    oz = _oz()
    m, n, k, phi, kbk, cut = case
    monkeypatch.setenv("OZ_PANEL_ROWS", "128")
    monkeypatch.setenv("OZ_PANEL_COLS", "96")
    rng = np.random.default_rng(m + n + k)
    A = spread_matrix(rng, m, k, phi)
    B = spread_matrix(rng, k, n, phi)
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), k_block=kbk, pair_cutoff=cut)
    res = oz.oz_gemm(A, B, cfg)
    Cref, info = oracle.oz_gemm(A, B, "fp8e4m3", "fp32", kbk, False, None, "smallest-first", cut)
    assert [(b.k_lo, b.k_hi, b.s_x, b.s_y) for b in res.stats.blocks] == info["blocks"]
    assert np.array_equal(bits(res.C), bits(Cref))


@pytest.mark.parametrize("kbk", [0, 96])
def test_host_output_overlapped_copy(cuda, kbk):
    """Host (pinned) inputs -> host C filled band by band while the GEMM runs
    (cuStreamWaitValue32 on per-band tile counters): bitwise the device result,
    several row bands, with and without k-blocking."""
    torch = cuda
    oz = _oz()
    rng = np.random.default_rng(4096)
    A = spread_matrix(rng, 4352, 256, 0.5)
    B = spread_matrix(rng, 256, 200, 0.5)
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), k_block=kbk)
    rd = oz.oz_gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), cfg)
    rh = oz.oz_gemm(torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory(), cfg)
    rn = oz.oz_gemm(A, B, cfg)
    assert not rh.C.is_cuda
    assert np.array_equal(bits(rh.C.numpy()), bits(rd.C.cpu().numpy()))
    assert np.array_equal(bits(rn.C), bits(rd.C.cpu().numpy()))


def test_fp6_formats(cuda):
    """FP6 slices: packed 6-bit planes through TMA 16U6_ALIGN16B into kind::f8f6f4
    E3M2 MMAs — fp6e3m2 slices and C bitwise equal to the oracle; fp6e2m3 fails the
    reference's way (SlicingInfeasible, slicing.py:169-172)."""
    import oracle

    oz = _oz()
    rng = np.random.default_rng(66)
    A = spread_matrix(rng, 300, 200, 0.5)
    B = spread_matrix(rng, 200, 136, 0.5)
    f = oz.get_format("fp6e3m2")
    params = oz.compute_params(53, f.mant_bits, 24, 200)
    ss = oz.slice_matrix(A, "rows", f, params)
    coeff, expo, _, s, flags = oracle.split_rows(A, params.rho, False)
    assert flags == 0 and ss.s == s
    for p in range(s):
        assert np.array_equal(bits(ss.coeff[p]), bits(coeff[p]))
    for kbk, emu in ((0, False), (64, False), (0, True)):
        res = oz.oz_gemm(A, B, oz.GemmConfig(f, oz.get_format("fp32"), k_block=kbk, fp64_emulation=emu))
        Cref, info = oracle.oz_gemm(A, B, "fp6e3m2", "fp32", kbk, emu)
        assert [(b.k_lo, b.k_hi, b.s_x, b.s_y) for b in res.stats.blocks] == info["blocks"]
        assert np.array_equal(bits(res.C), bits(Cref))
    with pytest.raises(oz.SlicingInfeasible):
        oz.oz_gemm(A, B, oz.GemmConfig(oz.get_format("fp6e2m3"), oz.get_format("fp32")))


def test_lp_gemm_fp6_exact(cuda):
    """The lp_gemm seam (lpgemm.py:93-120) with packed FP6 operands: exact."""
    oz = _oz()
    rng = np.random.default_rng(12)
    A = spread_matrix(rng, 130, 200, 0.5)
    B = spread_matrix(rng, 200, 70, 0.5)
    f = oz.get_format("fp6e3m2")
    params = oz.compute_params(53, f.mant_bits, 24, 200)
    sa = oz.slice_matrix(A, "rows", f, params)
    sb = oz.slice_matrix(B, "cols", f, params)
    for p in (0, sa.s - 1):
        for q in (0, sb.s - 1):
            G = oz.lp_gemm(oz.LpMatrix(sa.coeff[p], f), oz.LpMatrix(sb.coeff[q], f), oz.get_format("fp32"))
            assert np.array_equal(G, sa.coeff[p] @ sb.coeff[q])


FIXED_CASES = [
    # m, n, k, phi, type2, k_block, emu, max_slices, order, cutoff
    (128, 128, 128, 0.5, "fp8e4m3", 0, False, None, "smallest-first", None),
    (300, 260, 1000, 1.0, "fp8e4m3", 0, False, None, "smallest-first", 11),
    (257, 200, 700, 4.0, "fp8e4m3", 0, True, None, "smallest-first", 10),
    (200, 136, 640, 0.5, "fp8e4m3", 256, False, None, "largest-first", None),
    (129, 257, 333, 2.0, "fp8e4m3", 0, False, 6, "smallest-first", None),
    (256, 128, 512, 0.5, "fp16", 0, False, None, "smallest-first", 6),
    (160, 96, 700, 4.0, "fp16", 300, True, None, "smallest-first", None),
    (64, 64, 96, 1.0, "bf16", 0, False, None, "smallest-first", None),
]


@pytest.mark.parametrize("case", FIXED_CASES, ids=[f"{c[0]}x{c[1]}x{c[2]}-{c[4]}-kb{c[5]}-emu{int(c[6])}"
                                                   f"-ms{c[7]}-{c[8][:5]}-cut{c[9]}" for c in FIXED_CASES])
@pytest.mark.parametrize("variant", [("1", "64"), ("1", "128"), ("2", "128"), ("2", "192"), ("2", "256")],
                         ids=lambda v: f"cta{v[0]}-n{v[1]}")
def test_fixed_step_grouped_bitwise(cuda, case, variant, pair_variant):
    """slice_exponents="fixed" (opt-in): fixed-step slices and level-grouped
    tensor-core accumulation, bitwise against the CPU restatement
    (oracle.oz_gemm_fixed), in every kernel variant and both FP64 modes."""
    import oracle

    pair_variant(int(variant[0]), int(variant[1]))
    oz = _oz()
    m, n, k, phi, t2, kbk, emu, ms, order, cut = case
    rng = np.random.default_rng(m * 3 + n * 5 + k)
    A = spread_matrix(rng, m, k, phi)
    B = spread_matrix(rng, k, n, phi)
    cfg = oz.GemmConfig(oz.get_format(t2), oz.get_format("fp32"), k_block=kbk, fp64_emulation=emu,
                        max_slices=ms, accumulation_order=order, pair_cutoff=cut, slice_exponents="fixed")
    res = oz.oz_gemm(A, B, cfg)
    Cref, blocks = oracle.oz_gemm_fixed(A, B, t2, "fp32", kbk, ms, order, cut)
    assert [(b.k_lo, b.k_hi, b.s_x, b.s_y) for b in res.stats.blocks] == blocks
    nbad = int(np.sum(bits(res.C) != bits(Cref)))
    assert nbad == 0, f"{nbad}/{m * n} entries differ"


@pytest.mark.parametrize("fmt", ["fp8e4m3", "fp16"])
@pytest.mark.parametrize("emu", [False, True])
def test_fixed_step_split_bitwise(cuda, fmt, emu):
    """oz_split_fixed: slices and exponents (incl. the continued exponent
    sequence of padding planes) equal the CPU restatement; the slices
    reconstruct the input exactly."""
    import oracle
    from paper_2508_00441_b200.slicing import split_many_device

    torch = cuda
    oz = _oz()
    rng = np.random.default_rng(31)
    X = spread_matrix(rng, 90, 700, 3.0)
    X[5] = 0.0
    X[7, :] = 1.0  # a row that ends after one slice
    f = oz.get_format(fmt)
    params = oz.compute_params(53, f.mant_bits, 24, 700)
    (ds,), _ = split_many_device([torch.from_numpy(X).cuda()], f, params, emu, fixed=True)
    ss = oz.slicing.device_to_sliceset(ds, "rows", params)
    coeff, expo, cnt, s = oracle.split_rows_fixed(X, params.rho)
    assert ss.s == s
    for p in range(s):
        assert np.array_equal(bits(ss.coeff[p]), bits(coeff[p])), p
        assert np.array_equal(ss.expo[p], expo[p]), p
    rec = sum(np.ldexp(coeff[p], expo[p][:, None]) for p in range(s))
    assert np.array_equal(bits(rec), bits(X))


def _fixed_split_pair(torch, X, fmt, emu, max_planes, cols):
    """Split X's rows (cols=False) or the columns of X^T given as a transpose
    view (cols=True) with the fixed-step split and a plane limit."""
    from paper_2508_00441_b200.slicing import split_many_device, split_deferred

    oz = _oz()
    f = oz.get_format(fmt)
    params = oz.compute_params(53, f.mant_bits, 24, X.shape[1])
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    view = Xd.t().contiguous().t() if cols else Xd  # cols: same values, column-major storage
    (ds,), flags = split_many_device([view], f, params, emu, fixed=True, max_planes=max_planes)
    dd = split_deferred(view, f, params, emu, fixed=True, max_planes=max_planes)
    return ds, dd, flags, params


@pytest.mark.parametrize("fmt", ["fp8e4m3", "fp16", "fp6e3m2"])
@pytest.mark.parametrize("emu", [False, True])
@pytest.mark.parametrize("max_planes", [1, 5, 12, 40])
def test_fixed_split_plane_limit_rows_and_cols(cuda, fmt, emu, max_planes):
    """Fixed-step split with a plane limit (the barrier-free row path and the
    in-place column path, oz_split_fixed_cols): planes, exponents, counts and s
    equal the CPU restatement, for rows and for columns read in place, through
    both the synchronous and the deferred (sync-free) split."""
    import oracle

    torch = cuda
    rng = np.random.default_rng(77 + max_planes)
    X = spread_matrix(rng, 70, 1100, 3.0)
    X[5] = 0.0
    X[7, :] = 1.0            # ends after one slice
    X[9, 3] = 2.0 ** -1000   # tiny input: checked slicing
    X[11, :] *= 2.0 ** 600
    coeff, expo, cnt, s = oracle.split_rows_fixed(X, _oz().compute_params(53, _oz().get_format(fmt).mant_bits, 24,
                                                                          X.shape[1]).rho, max_planes)
    for cols in (False, True):
        ds, dd, flags, params = _fixed_split_pair(torch, X, fmt, emu, max_planes, cols)
        assert flags == 0
        assert ds.s == s, (cols, ds.s, s)
        assert np.array_equal(ds.row_cnt.cpu().numpy(), cnt), cols
        ss = _oz().slicing.device_to_sliceset(ds, "rows", params)
        for p in range(s):
            assert np.array_equal(bits(ss.coeff[p]), bits(coeff[p])), (cols, p)
            assert np.array_equal(ss.expo[p], expo[p]), (cols, p)
        sf = dd.sf.cpu().tolist()
        if max_planes > 32:  # deferred: cap = 32 planes, the caller redoes the split
            assert sf[1] == 256, (cols, sf)
            continue
        assert sf[0] == s and sf[1] == 0, (cols, sf)
        codes_d = dd.codes()[:s].cpu().numpy()
        assert np.array_equal(codes_d, ds.codes()[:s].cpu().numpy()), cols
        assert np.array_equal(dd.row_cnt.cpu().numpy(), cnt), cols


@pytest.mark.parametrize("emu", [False, True])
def test_fixed_cols_split_matches_transpose(cuda, emu):
    """oz_split_fixed_cols on B[lo:hi, j0:j1] (strided, odd sizes, a panel
    offset) is bitwise the transpose + row split the reference-order path uses."""
    from paper_2508_00441_b200.slicing import split_many_device, transpose_device

    torch = cuda
    oz = _oz()
    rng = np.random.default_rng(5)
    B = torch.from_numpy(spread_matrix(rng, 777, 301, 2.0)).cuda()
    Bv = B[33:700, 17:290]
    f = oz.get_format("fp8e4m3")
    params = oz.compute_params(53, f.mant_bits, 24, Bv.shape[0])
    (dc,), fc = split_many_device([Bv.t()], f, params, emu, fixed=True, max_planes=11)
    (dt,), ft = split_many_device([transpose_device(Bv)], f, params, emu, fixed=True, max_planes=11)
    assert fc == ft == 0 and dc.s == dt.s
    assert torch.equal(dc.codes()[:dc.s], dt.codes()[:dt.s])
    assert torch.equal(dc.expo[:dc.s], dt.expo[:dt.s])
    assert torch.equal(dc.row_cnt, dt.row_cnt)


def test_fixed_cols_split_errors(cuda):
    """Non-finite and subnormal inputs in a column raise like the reference
    (ValueError / RangeError) through the in-place column split."""
    oz = _oz()
    rng = np.random.default_rng(9)
    A = spread_matrix(rng, 64, 300, 0.5)
    for bad, exc in ((np.nan, ValueError), (np.inf, ValueError), (5e-324, oz.RangeError)):
        B = spread_matrix(rng, 300, 80, 0.5)
        B[100, 41] = bad
        cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), pair_cutoff=9, slice_exponents="fixed")
        with pytest.raises(exc):
            oz.oz_gemm(A, B, cfg)


@pytest.mark.parametrize("kw", [{}, {"pair_cutoff": 9, "slice_exponents": "fixed"}, {"k_block": 256},
                                {"fp64_emulation": True}, {"type2": "fp16", "k_block": 300}],
                         ids=["defaults", "fixed9", "kb256", "emu", "fp16kb300"])
def test_graph_replay_bitwise(cuda, kw):
    """oz_gemm_device(graph=True): the captured CUDA graph, replayed on new
    contents of the same operand buffers, gives bitwise the eager C, and a
    non-finite input written after the capture still raises ValueError."""
    torch = cuda
    oz = _oz()
    kw = dict(kw)
    t2 = kw.pop("type2", "fp8e4m3")
    cfg = oz.GemmConfig(oz.get_format(t2), oz.get_format("fp32"), **kw)
    rng = np.random.default_rng(3)
    A = torch.from_numpy(spread_matrix(rng, 300, 700, 1.0)).cuda()
    B = torch.from_numpy(spread_matrix(rng, 700, 260, 1.0)).cuda()
    Cg = torch.empty((300, 260), dtype=torch.float64, device="cuda")
    for it in range(3):
        A.copy_(torch.from_numpy(spread_matrix(rng, 300, 700, 0.5 + it)))
        B.copy_(torch.from_numpy(spread_matrix(rng, 700, 260, 0.5 + it)))
        _, sg = oz.oz_gemm_device(A, B, cfg, out=Cg, graph=True)
        Ce, se = oz.oz_gemm_device(A, B, cfg)
        assert torch.equal(Cg.view(torch.int64), Ce.view(torch.int64)), it
        assert [(b.s_x, b.s_y) for b in sg.blocks] == [(b.s_x, b.s_y) for b in se.blocks]
        assert sg.t_gemm > 0
    A[5, 7] = float("nan")
    with pytest.raises(ValueError):
        oz.oz_gemm_device(A, B, cfg, out=Cg, graph=True)


@pytest.mark.parametrize("kw", [{}, {"fp64_emulation": True}, {"pair_cutoff": 9, "slice_exponents": "fixed"},
                                {"k_block": 512}], ids=["defaults", "emu", "fixed9", "kb512"])
def test_variants_agree_multiwave(cuda, kw, pair_variant):
    """Every kernel variant (1-CTA 128x64 and 128x128, CTA-pair 256x128 and
    256x192) over several persistent-tile waves gives bitwise the same C."""
    torch = cuda
    oz = _oz()
    rng = np.random.default_rng(21)
    A = torch.from_numpy(spread_matrix(rng, 2048, 1024, 1.0)).cuda()
    B = torch.from_numpy(spread_matrix(rng, 1024, 1920, 1.0)).cuda()
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), **kw)
    ref = None
    for cta, tn in ((2, 192), (1, 64), (1, 128), (2, 128)):
        if kw.get("fp64_emulation") and tn == 192:
            continue
        pair_variant(cta, tn)
        C, _ = oz.oz_gemm_device(A, B, cfg)
        if ref is None:
            ref = C.clone()
        else:
            assert torch.equal(C.view(torch.int64), ref.view(torch.int64)), (cta, tn)


@pytest.mark.parametrize("shape", [(1100, 1300, 1000), (600, 515, 333)], ids=["multiwave", "ragged"])
def test_fixed_step_wide_tiles_bitwise(cuda, shape, pair_variant):
    """256 x 256 CTA-pair tiles (fixed-step grouped mode; half of Cb read-modify-
    written in C itself): bitwise the CPU restatement over several tile waves,
    ragged edges, and 128-row slabs whose A slices are all zero (every group
    of that CTA skipped: its C-resident columns must still be written as +0)."""
    import oracle

    pair_variant(2, 256)
    oz = _oz()
    m, n, k = shape
    rng = np.random.default_rng(m + n + k)
    A = spread_matrix(rng, m, k, 1.0)
    A[128:256] = 0.0  # one whole 128-row slab of zeros
    A[300, :] *= 2.0 ** 40
    B = spread_matrix(rng, k, n, 1.0)
    for cut in (11, 6):
        cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), pair_cutoff=cut,
                            slice_exponents="fixed")
        res = oz.oz_gemm(A, B, cfg)
        Cref, _ = oracle.oz_gemm_fixed(A, B, "fp8e4m3", "fp32", 0, None, "smallest-first", cut)
        nbad = int(np.sum(bits(res.C) != bits(Cref)))
        assert nbad == 0, f"cut {cut}: {nbad}/{m * n} entries differ"


@pytest.mark.parametrize("kw", [{}, {"pair_cutoff": 9, "slice_exponents": "fixed"}, {"fp64_emulation": True}],
                         ids=["defaults", "fixed9", "emu"])
def test_tuning_knobs_keep_bits(cuda, kw):
    """oz_set_epilogue_warps(12) (N = 192 kernel) and oz_set_pair_schedule(1)
    (exclusive epilogue windows) change scheduling only: C is bitwise the
    default over several tile waves."""
    from paper_2508_00441_b200 import _lib

    torch = cuda
    oz = _oz()
    rng = np.random.default_rng(8)
    A = torch.from_numpy(spread_matrix(rng, 1500, 1024, 1.0)).cuda()
    B = torch.from_numpy(spread_matrix(rng, 1024, 2100, 1.0)).cuda()
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), **kw)
    ref, _ = oz.oz_gemm_device(A, B, cfg)
    try:
        for warps, sched in ((12, 0), (8, 1), (12, 1)):
            _lib.call("oz_set_epilogue_warps", warps)
            _lib.call("oz_set_pair_schedule", sched)
            C, _ = oz.oz_gemm_device(A, B, cfg)
            assert torch.equal(C.view(torch.int64), ref.view(torch.int64)), (warps, sched)
    finally:
        _lib.call("oz_set_epilogue_warps", 8)
        _lib.call("oz_set_pair_schedule", 0)


def _structured_rows(rng, rows, kb):
    """Rows whose slice exponents do not follow c_p = c_0 - p (54 - rho) (a
    residual max below a quarter of the grid step, early ends, single elements)
    mixed with random rows."""
    X = spread_matrix(rng, rows, kb, 1.0)
    X[0] = 1.0                                   # ends after one slice
    X[1] = 1.0 + 2.0 ** -30                      # residual 2^-30: mismatch at slice 1
    X[2] = 0.0
    X[2, kb // 2] = -3.0 + 2.0 ** -40            # single element
    X[3] = rng.integers(-7, 8, kb).astype(np.float64) * (1.0 + 2.0 ** -22 + 2.0 ** -47)
    X[4] = np.ldexp(1.0, rng.integers(-20, 20, kb))  # powers of two over a range
    X[5] = (1.0 + 2.0 ** -20 + 2.0 ** -45) * np.sign(rng.standard_normal(kb))
    X[6, ::3] = 2.0 ** -35                       # small entries next to random ones
    X[7] = np.where(rng.random(kb) < 0.01, rng.standard_normal(kb), 0.0)  # sparse
    return X


@pytest.mark.parametrize("fmt", ["fp8e4m3", "fp16", "bf16", "fp6e3m2"])
@pytest.mark.parametrize("emu", [False, True])
@pytest.mark.parametrize("kb", [37, 4096, 8192, 20000])
def test_split_structured_rows(cuda, fmt, emu, kb):
    """Adaptive row split on structured rows (early ends, residual maxima far
    below the grid step so exponents jump, single elements, powers of two,
    sparse rows) at every launch shape (kb up to 4096, the 256 x 32 / 512 x 16
    rows, 4-CTA clusters), hardware and emulated (fixed-point residuals): the
    reference's slices, exponents and counts."""
    import oracle

    oz = _oz()
    rng = np.random.default_rng(kb + 7 * emu)
    X = _structured_rows(rng, 12, kb)
    params = oz.compute_params(53, oz.get_format(fmt).mant_bits, 24, kb)
    ss = oz.slice_matrix(X, "rows", oz.get_format(fmt), params, "emu" if emu else "fp64")
    coeff, expo, cnt, s, flags = oracle.split_rows(X, params.rho, emu)
    assert flags == 0 and ss.s == s
    for p in range(s):
        assert np.array_equal(bits(ss.coeff[p]), bits(coeff[p])), f"coeff plane {p}"
        assert np.array_equal(ss.expo[p], expo[p].astype(np.int64)), f"expo plane {p}"


@pytest.mark.parametrize("emu", [False, True])
def test_oz_gemm_structured_rows_bitwise(cuda, emu):
    import oracle

    oz = _oz()
    rng = np.random.default_rng(99)
    A = _structured_rows(rng, 130, 700)
    B = _structured_rows(rng, 140, 700).T.copy()
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), fp64_emulation=emu)
    C = oz.oz_gemm(A, B, cfg).C
    Cref, _ = oracle.oz_gemm(A, B, "fp8e4m3", "fp32", 0, emu)
    assert np.array_equal(bits(C), bits(Cref))





@pytest.mark.parametrize("fixed", [False, True])
def test_emulated_split_fixed_point_rows(cuda, fixed):
    """Emulated row split at kb = 8192 (fixed-point residuals: fx_state/fx_slice,
    keys from fx_key), adaptive and fixed-step: slices, exponents and counts are
    the oracle's, incl. structured rows and a row whose elements span too many
    binades for the fixed-point shift field (that thread keeps FP64 words)."""
    import oracle

    torch = cuda
    oz = _oz()
    rng = np.random.default_rng(5 + fixed)
    X = _structured_rows(rng, 40, 8192)
    X[20, 5] = 2.0 ** 400
    X[20, 6] = 2.0 ** -600
    f = oz.get_format("fp8e4m3")
    params = oz.compute_params(53, f.mant_bits, 24, 8192)
    if fixed:
        ds, _, flags, _ = _fixed_split_pair(torch, X, "fp8e4m3", True, 12, False)
        coeff, expo, cnt, s = oracle.split_rows_fixed(X, params.rho, 12)
        assert flags == 0 and ds.s == s
        assert np.array_equal(ds.row_cnt.cpu().numpy(), cnt)
        ss = oz.slicing.device_to_sliceset(ds, "rows", params)
    else:
        ss = oz.slice_matrix(X, "rows", f, params, "emu")
        coeff, expo, _, s, flags = oracle.split_rows(X, params.rho, True)
        assert flags == 0 and ss.s == s
    for p in range(s):
        assert np.array_equal(bits(ss.coeff[p]), bits(coeff[p])), f"coeff plane {p}"
        assert np.array_equal(np.asarray(ss.expo[p]), np.asarray(expo[p]).astype(np.int64)), f"expo plane {p}"


@pytest.mark.parametrize("t2,kbk", [("fp8e4m3", 0), ("fp8e5m2", 0), ("bf16", 256), ("fp6e3m2", 0)])
def test_type3_fp64_within_exact_range(cuda, t2, kbk):
    """type3 = fp64 (the reference accumulates lp_gemm in FP64, per-step RNE):
    wherever every partial sum of a k-block fits the FP32 tensor-core
    accumulator exactly (kb <= 2^(24 - 2 (53 - rho))), both accumulations are
    exact, so C is the reference's bit for bit."""
    import oracle

    oz = _oz()
    rng = np.random.default_rng(64)
    A = spread_matrix(rng, 150, 600, 1.0)
    B = spread_matrix(rng, 600, 130, 1.0)
    cfg = oz.GemmConfig(oz.get_format(t2), oz.get_format("fp64"), k_block=kbk)
    res = oz.oz_gemm(A, B, cfg)
    Cref, info = oracle.oz_gemm(A, B, t2, "fp64", kbk, False)
    assert info["flags"] == 0
    assert [(b.k_lo, b.k_hi, b.s_x, b.s_y) for b in res.stats.blocks] == info["blocks"]
    assert np.array_equal(bits(res.C), bits(Cref))


def test_type3_fp64_beyond_exact_range_raises(cuda):
    """FP16 slices with type3 = fp64 get rho = 42 (11-bit digits): a k-block of
    600 would need 35-bit partial sums — not available on the tensor cores, so
    the call raises instead of returning a differently rounded C."""
    oz = _oz()
    rng = np.random.default_rng(65)
    A = spread_matrix(rng, 64, 600, 1.0)
    B = spread_matrix(rng, 600, 64, 1.0)
    with pytest.raises(NotImplementedError):
        oz.oz_gemm(A, B, oz.GemmConfig(oz.get_format("fp16"), oz.get_format("fp64")))


@pytest.mark.parametrize("variant", [("1", "64"), ("1", "128"), ("2", "128"), ("2", "192"), ("2", "256")],
                         ids=lambda v: f"cta{v[0]}-n{v[1]}")
@pytest.mark.parametrize("fixed", [False, True])
def test_production_accumulator_is_exact_ladder(cuda, variant, fixed, pair_variant):
    """K4 on the production kernels (regression for profiles/accwidth_r01.json,
    which probed the lp_gemm tile kernel): C[r, r] = 2^r unit products + one
    product of two grid minima (2^-4 * 2^-4) must come out as 2^r + 2^-8
    exactly for r up to 15 (24 significant bits, the FP8 k-block bound
    kb <= 2^16).  Every operand is one slice (digits 16 and 1 on the 2^-4 grid),
    so C = G of the single pair: any truncation inside the tcgen05 FP32
    accumulation would show, in every kernel variant the planner can pick."""
    if variant[1] == "256" and not fixed:
        pytest.skip("256-column tiles are a fixed-step variant")
    pair_variant(int(variant[0]), int(variant[1]))
    oz = _oz()
    R, k = 16, (1 << 15) + 128
    A = np.zeros((R, k))
    B = np.zeros((k, R))
    for r in range(R):
        A[r, : 1 << r] = 1.0
        B[: 1 << r, r] = 1.0
        A[r, k - 1 - r] = 2.0 ** -4
        B[k - 1 - r, r] = 2.0 ** -4
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"),
                        slice_exponents="fixed" if fixed else "adaptive")
    res = oz.oz_gemm(A, B, cfg)
    assert [(b.s_x, b.s_y) for b in res.stats.blocks] == [(1, 1)]
    want = np.array([2.0 ** r + 2.0 ** -8 for r in range(R)])
    assert np.array_equal(np.diag(res.C), want), np.diag(res.C) - want
