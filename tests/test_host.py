"""Host-side logic (no GPU): slicing constants, GEMM-count planning, config
validation, exception classes, pair order, format codecs — checked against
the reference's golden vectors."""

import itertools
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2508_00441_b200 as oz
from paper_2508_00441_b200.formats import decode_codes
from paper_2508_00441_b200.lpgemm import encode_values
from paper_2508_00441_b200.ozgemm import pair_order

GOLD = Path(__file__).resolve().parent / "golden"
PARAMS = json.loads((GOLD / "params.json").read_text())
ERRORS = json.loads((GOLD / "errors.json").read_text())


@pytest.mark.parametrize("kat", PARAMS["kats"], ids=lambda d: f"m2={d['m2']}-m3={d['m3']}-k={d['k']}")
def test_compute_params_kats(kat):
    p = oz.compute_params(53, kat["m2"], kat["m3"], kat["k"])
    assert (p.gamma, p.xi, p.rho, p.slice_width, p.feasible) == (
        kat["gamma"], kat["xi"], kat["rho"], kat["width"], kat["feasible"])
    assert oz.predict_slice_count(p) == kat["pred_s"]
    assert oz.predict_gemm_count(53, kat["m2"], kat["m3"], kat["k"]) == kat["pred_g"]


def test_gemm_count_table_matches_reference():
    for row in PARAMS["table"]:
        got = oz.predict_gemm_count(53, oz.FORMATS[row["type2"]].mant_bits, oz.FORMATS[row["type3"]].mant_bits,
                                    row["k"])
        assert got == row["count"], row


def test_paper_table_spot_values():
    # PAPER.md:238-265 / SPEC acceptance: FP8/FP32 -> 121, FP16/FP32 @ 8192 -> 81
    assert oz.predict_gemm_count(53, 4, 24, 65536) == 121
    assert oz.predict_gemm_count(53, 11, 24, 8192) == 81
    assert not oz.compute_params(53, 11, 11, 4096).feasible


def test_oz_gemm_count_blocked():
    f16, f32 = oz.get_format("fp16"), oz.get_format("fp32")
    cfg = oz.GemmConfig(f16, f32, k_block=4096)
    assert oz.oz_gemm_count(16384, 16384, 16384, cfg) == 4 * oz.predict_gemm_count(53, 11, 24, 4096)
    with pytest.raises(oz.SlicingInfeasible):
        oz.oz_gemm_count(64, 64, 4096, oz.GemmConfig(f16, oz.get_format("fp16")))


@pytest.mark.parametrize("name,kw", [("kblock_neg", {"k_block": -1}), ("max_slices0", {"max_slices": 0}),
                                     ("bad_order", {"accumulation_order": "random"})])
def test_config_validation_matches_reference(name, kw):
    assert ERRORS[name][0] == "ValueError"  # what the reference raised
    with pytest.raises(ValueError):
        oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), **kw)


def test_exception_hierarchy_matches_reference():
    assert issubclass(oz.RangeError, ArithmeticError)
    assert issubclass(oz.DimensionError, ValueError)
    assert issubclass(oz.SlicingInfeasible, Exception) and not issubclass(oz.SlicingInfeasible, ValueError)
    for name in ("subnormal_input", "shape_mismatch"):
        mro = ERRORS[name][1]
        cls = getattr(oz, mro[0])
        assert [c.__name__ for c in cls.__mro__] == mro


def test_formats_catalog():
    assert set(oz.FORMATS) == {"fp16", "bf16", "fp8e4m3", "fp8e5m2", "fp6e3m2", "fp6e2m3", "fp32", "fp64"}
    assert oz.get_format("FP8E4M3").max_finite == 448.0
    assert oz.get_format("fp16").mant_bits == 11 and oz.get_format("bf16").mant_bits == 8
    with pytest.raises(ValueError):
        oz.get_format("fp7")


@pytest.mark.parametrize("sx,sy", [(1, 1), (3, 5), (17, 17), (24, 23), (5, 2)])
@pytest.mark.parametrize("order", ["smallest-first", "largest-first"])
def test_pair_order_is_reference_sort(sx, sy, order):
    ref = sorted(itertools.product(range(sx), range(sy)),
                 key=(lambda pq: (-(pq[0] + pq[1]), pq[0], pq[1])) if order == "smallest-first"
                 else (lambda pq: (pq[0] + pq[1], pq[0], pq[1])))
    assert pair_order(sx, sy, order) == ref
    for d in (0, 3, sx + sy - 2):
        assert pair_order(sx, sy, order, d) == [pq for pq in ref if sum(pq) <= d]


def _pair_iter(lp, lq, order, cutoff):
    """Python transcription of PairIter (oz_pair_gemm.cu) to test the device enumeration."""
    out = []
    dmax = lp + lq - 2
    if cutoff >= 0 and cutoff < dmax:
        dmax = cutoff
    if lp <= 0 or lq <= 0:
        return out
    d = dmax if order == 0 else 0
    step = -1 if order == 0 else 1
    while 0 <= d <= dmax:
        for p in range(max(0, d - (lq - 1)), min(d, lp - 1) + 1):
            out.append((p, d - p))
        d += step
    return out


@pytest.mark.parametrize("lp,lq", [(1, 1), (2, 7), (17, 17), (9, 3), (0, 4)])
@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("cutoff", [-1, 0, 5, 12])
def test_device_pair_enumeration_is_subsequence(lp, lq, order, cutoff):
    want = pair_order(lp, lq, "smallest-first" if order == 0 else "largest-first",
                      None if cutoff < 0 else cutoff)
    assert _pair_iter(lp, lq, order, cutoff) == want


@pytest.mark.parametrize("fmt", ["fp8e4m3", "fp8e5m2", "fp16", "bf16"])
def test_codec_roundtrip(fmt):
    f = oz.get_format(fmt)
    rng = np.random.default_rng(0)
    params = oz.compute_params(53, f.mant_bits, 24, 4096)
    q = 2.0 ** (params.rho - 53)
    lim = int(round(1 / q))
    vals = rng.integers(-lim, lim + 1, size=(64, 64)) * q
    codes = encode_values(vals, f)
    assert np.array_equal(decode_codes(codes, fmt), vals)
    with pytest.raises(oz.RepresentabilityError):
        encode_values(np.array([[q / 3]]), f)


def test_backend_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"))
    with pytest.raises(oz.BackendUnavailable):
        oz.oz_gemm(np.ones((2, 2)), np.ones((2, 2)), cfg)


class _FakeCuda:
    """Just enough of torch.cuda for the panel planner (no GPU)."""

    def __init__(self, total_gib, free_gib):
        self.total, self.free = total_gib << 30, free_gib << 30

    def current_device(self):
        return 0

    def get_device_properties(self, d):
        return type("P", (), {"total_memory": self.total})

    def mem_get_info(self):
        return self.free, self.total

    def memory_reserved(self, d=None):  # nothing cached by the allocator
        return 0

    def memory_allocated(self, d=None):
        return 0


def test_panel_plan_small_problems_unpanelled():
    from paper_2508_00441_b200 import ozgemm

    ozgemm._TOTAL_MEM.clear()
    torch = type("T", (), {"cuda": _FakeCuda(178, 170)})
    for n in (128, 1024, 8192, 16384):
        assert ozgemm._panel_plan(n, n, n, 1, torch) == (n, n)


def test_panel_plan_n65536_one_gpu_fits():
    """n = 65536 FP8 next to 96 GiB of FP64 operands: panels whose slice buffers fit."""
    from paper_2508_00441_b200 import ozgemm
    from paper_2508_00441_b200.slicing import PLANE_CAP, _plane_cap

    ozgemm._TOTAL_MEM.clear()
    torch = type("T", (), {"cuda": _FakeCuda(178, 178 - 96)})
    n = 65536
    mp, np_ = ozgemm._panel_plan(n, n, n, 1, torch)
    assert mp < n and np_ < n and n % mp == 0 and n % np_ == 0
    ld = n
    need = 8 * n * np_ + max(_plane_cap(np_, ld, 15), 24) * np_ * ld + max(_plane_cap(mp, ld, 15), 24) * mp * ld
    assert need <= (178 - 96 - 6) << 30
    assert PLANE_CAP >= 24


def test_fp64_level_summary_picks_fastest_accurate_variant():
    import bench

    extras = {"accuracy": {"max_rel_err_ozaki": 8e-12, "max_rel_err_cublas_dgemm": 3e-9},
              "native_dgemm": {"tflops": 35.0},
              "variants": {"fp8_pair_cutoff_12": {"tflops": 26.0, "max_rel_err": 8e-12},
                           "fp8_pair_cutoff_11": {"tflops": 30.0, "max_rel_err": 4e-10},
                           "fp8_pair_cutoff_10": {"tflops": 36.0, "max_rel_err": 4e-9},
                           "fp8_emulated_fp64": {"tflops": 6.0, "max_rel_err": 8e-12}}}
    s = bench.fp64_level_summary(extras)
    assert s["config"].startswith("pair_cutoff_11") and s["tflops"] == 30.0
    assert abs(s["vs_native_dgemm"] - 30.0 / 35.0) < 1e-12
    assert bench.fp64_level_summary({}) is None


def test_fp6_pack_unpack_roundtrip():
    """Host packer (lp_gemm seam) and unpacker (slice decode) of the dense FP6 layout."""
    from paper_2508_00441_b200.lpgemm import _pack_fp6
    from paper_2508_00441_b200.slicing import unpack_fp6

    c = np.random.default_rng(1).integers(0, 64, size=(5, 256)).astype(np.uint8)
    packed = _pack_fp6(c)
    assert packed.shape == (5, 192)
    assert np.array_equal(unpack_fp6(packed), c)
    # bit order: code j of a group occupies bits [6j, 6j+6) little-endian
    one = np.zeros((1, 16), np.uint8)
    one[0, 10] = 63
    v = int.from_bytes(_pack_fp6(one)[0].tobytes(), "little")
    assert v == 63 << 60


def test_lp_gemm_refuses_products_whose_accumulation_can_round():
    """lp_gemm is the exact-product seam: operands whose per-step type3
    accumulation could round (lpgemm.py:49-77) raise instead of returning an
    FP32-accumulated result that could differ from the reference."""
    from paper_2508_00441_b200 import LpMatrix, get_format, lp_gemm
    from paper_2508_00441_b200.lpgemm import accumulation_is_exact

    f16, f32, e4m3 = get_format("fp16"), get_format("fp32"), get_format("fp8e4m3")
    A = np.array([[1.0, 2.0 ** -13]])
    B = np.array([[1.0], [1.0]])
    assert accumulation_is_exact(A, B, f32) and not accumulation_is_exact(A, B, f16)
    with pytest.raises(NotImplementedError):
        lp_gemm(LpMatrix(A, f16), LpMatrix(B, f16), f16)
    # 2^-12 * 2^-12 products next to 1.0: 25 bits, too wide for FP32
    A = np.array([[1.0, 2.0 ** -12]])
    B = np.array([[1.0], [2.0 ** -12]])
    assert not accumulation_is_exact(A, B, f32)
    with pytest.raises(NotImplementedError):
        lp_gemm(LpMatrix(A, f16), LpMatrix(B, f16), f32)
    # slice-like operands on the 2^-4 grid, k = 4096: exact
    rng = np.random.default_rng(0)
    A = rng.integers(-16, 17, size=(3, 4096)) / 16.0
    B = rng.integers(-16, 17, size=(4096, 2)) / 16.0
    assert accumulation_is_exact(A, B, f32)
    assert not accumulation_is_exact(A * 1024, B * 1024, get_format("fp16"))
    assert accumulation_is_exact(np.zeros((2, 2)), B[:2], e4m3)


def test_panel_plan_counts_cached_allocator_memory():
    """Blocks torch's caching allocator holds but has not handed out count as
    free (with them ignored, n = 65536 on one GPU degraded to tiny panels)."""
    from paper_2508_00441_b200 import ozgemm

    class _Cached(_FakeCuda):
        def memory_reserved(self, d=None):
            return 60 << 30

        def memory_allocated(self, d=None):
            return 0

    ozgemm._TOTAL_MEM.clear()
    n = 65536
    bare = ozgemm._panel_plan(n, n, n, 1, type("T", (), {"cuda": _FakeCuda(178, 178 - 96 - 60)}))
    cached = ozgemm._panel_plan(n, n, n, 1, type("T", (), {"cuda": _Cached(178, 178 - 96 - 60)}))
    assert cached[0] * cached[1] > bare[0] * bare[1]
    assert cached == ozgemm._panel_plan(n, n, n, 1, type("T", (), {"cuda": _FakeCuda(178, 178 - 96)}))
