"""One slice-pair product on the tensor cores — the ``lp_gemm`` seam.

The reference simulates a low-precision GEMM with per-step RNE accumulation
in numpy (lpgemm.py:93-120).  Here the operands are real FP8/FP16 codes fed
to one tcgen05 MMA tile kernel (``oz_lp_gemm``) with FP32 accumulation in
TMEM.  For slice operands the product is exact (error-free by construction),
so the result equals the reference's bit for bit; that is the only regime the
pipeline uses.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import RepresentabilityError
from .formats import FormatSpec, decode_codes

__all__ = ["RepresentabilityError", "LpMatrix", "lp_gemm", "encode_values"]


class LpMatrix:
    """Matrix whose entries are representable in ``fmt`` (lpgemm.py:27-46)."""

    def __init__(self, data, fmt: FormatSpec, _validated: bool = False):
        self.data = np.asarray(data, dtype=np.float64)
        self.fmt = fmt
        if self.data.ndim != 2:
            raise ValueError("LpMatrix expects a 2-D matrix")
        if not _validated:
            encode_values(self.data, fmt)  # raises RepresentabilityError

    @property
    def shape(self):
        return self.data.shape


def encode_values(vals: np.ndarray, fmt: FormatSpec) -> np.ndarray:
    """Exact float64 values -> storage codes (uint8 / uint16); raises
    RepresentabilityError for a value the format cannot hold exactly."""
    vals = np.asarray(vals, dtype=np.float64)
    if fmt.name in ("fp8e4m3", "fp8e5m2", "fp6e3m2", "fp6e2m3"):
        table = decode_codes(np.arange(256, dtype=np.uint8), fmt.name)
        ok = np.isfinite(table)
        if fmt.name == "fp8e4m3":
            ok &= np.arange(256) & 0x7F != 0x7F  # S.1111.111 is NaN
        elif fmt.name == "fp8e5m2":
            ok &= (np.arange(256) >> 2) & 0x1F != 0x1F
        else:  # FP6: only canonical containers (the code at FP6_SHIFT, other bits 0)
            from .formats import FP6_SHIFT

            ok &= (np.arange(256) & ~(63 << FP6_SHIFT)) == 0
        codes_ok = np.nonzero(ok)[0]
        vals_ok = table[codes_ok]
        order = np.argsort(vals_ok, kind="stable")
        sv, sc = vals_ok[order], codes_ok[order]
        idx = np.clip(np.searchsorted(sv, vals), 0, sv.size - 1)
        if not np.all(sv[idx] == vals):
            raise RepresentabilityError(f"matrix entries not representable in {fmt.name}")
        out = sc[idx].astype(np.uint8)
        out[vals == 0] = 0
        return out
    if fmt.name == "fp16":
        h = vals.astype(np.float16)
        if not np.array_equal(h.astype(np.float64), vals):
            raise RepresentabilityError(f"matrix entries not representable in {fmt.name}")
        return h.view(np.uint16)
    if fmt.name == "bf16":
        f = vals.astype(np.float32)
        bits = f.view(np.uint32)
        if not np.array_equal(f.astype(np.float64), vals) or np.any(bits & 0xFFFF):
            raise RepresentabilityError(f"matrix entries not representable in {fmt.name}")
        return (bits >> 16).astype(np.uint16)
    raise NotImplementedError(f"no tensor-core operand path for {fmt.name} in this build")  # not reached for FP6


def _pack_fp6(codes: np.ndarray) -> np.ndarray:
    """[rows, ld] 6-bit codes (ld a multiple of 16) -> [rows, ld*3/4] bytes, 16
    codes per 12 bytes little-endian (the global side of TMA 16U6_ALIGN16B)."""
    g = codes.reshape(codes.shape[0], -1, 16).astype(np.uint64)
    lo = np.zeros(g.shape[:2], dtype=np.uint64)
    hi = np.zeros(g.shape[:2], dtype=np.uint64)
    for j in range(16):
        b = 6 * j
        v = g[..., j] & np.uint64(63)
        if b < 64:
            lo |= v << np.uint64(b)  # (bits past 63 fall off)
        if b >= 64:
            hi |= v << np.uint64(b - 64)
        elif b + 6 > 64:  # straddles the two words
            hi |= v >> np.uint64(64 - b)
    out = np.empty(g.shape[:2] + (12,), dtype=np.uint8)
    for i in range(8):
        out[..., i] = ((lo >> np.uint64(8 * i)) & np.uint64(255)).astype(np.uint8)
    for i in range(4):
        out[..., 8 + i] = ((hi >> np.uint64(8 * i)) & np.uint64(255)).astype(np.uint8)
    return out.reshape(codes.shape[0], -1)


def _padded_codes(torch, codes: np.ndarray, fp6: bool = False):
    rows, k = codes.shape
    if fp6:  # packed FP6 rows: ld a multiple of 128 codes
        ld = -(-max(k, 1) // 128) * 128
        buf = np.zeros((rows, ld), dtype=np.uint8)
        buf[:, :k] = codes
        return torch.from_numpy(_pack_fp6(buf)).cuda(), ld
    per16 = 16 // codes.itemsize
    ld = -(-max(k, 1) // per16) * per16
    buf = np.zeros((rows, ld), dtype=codes.dtype)
    buf[:, :k] = codes
    t = torch.from_numpy(buf.view(np.uint8) if codes.itemsize == 1 else buf.view(np.int16)).cuda()
    return t, ld


def _lsb_exponent(M: np.ndarray):
    """Smallest exponent e with every non-zero entry a multiple of 2^e, and the
    largest magnitude (None, 0 for an all-zero matrix)."""
    v = np.abs(M[M != 0])
    if v.size == 0:
        return None, 0.0
    bits = v.view(np.uint64)
    field = (bits >> np.uint64(52)).astype(np.int64)
    sig = (bits & np.uint64((1 << 52) - 1)) | np.where(field > 0, np.uint64(1 << 52), np.uint64(0))
    tz = np.zeros(sig.shape, dtype=np.int64)
    s = sig.copy()
    for sh in (32, 16, 8, 4, 2, 1):  # count trailing zeros of the significand
        low = (s & np.uint64((1 << sh) - 1)) == 0
        tz += np.where(low, sh, 0)
        s = np.where(low, s >> np.uint64(sh), s)
    return int(np.min(np.maximum(field, 1) - 1075 + tz)), float(v.max())


def accumulation_is_exact(A: np.ndarray, B: np.ndarray, type3: FormatSpec) -> bool:
    """True when every partial sum of A @ B, in any order, is exactly
    representable both in type3 and in the tensor cores' FP32 accumulator.
    Then the reference's per-step type3 RNE accumulation (lpgemm.py:49-77,
    105-119) and tcgen05's FP32 accumulation both produce the exact product, so
    they agree bit for bit.  All products are multiples of 2^(ga + gb) and every
    partial sum is bounded by k * max|A| * max|B|."""
    k = A.shape[1]
    ga, ma = _lsb_exponent(A)
    gb, mb = _lsb_exponent(B)
    if ga is None or gb is None or k == 0:
        return True
    g = ga + gb
    bound = k * ma * mb
    width = min(type3.mant_bits, 24)
    return (bound <= 2.0 ** (g + width)           # N * 2^g with |N| <= 2^m3 fits the significand
            and g >= type3.exp_min - type3.mant_bits + 1 and g >= -126  # grid above the subnormal quantum
            and bound <= type3.max_finite and bound < 2.0 ** 127)


def lp_gemm(A: LpMatrix, B: LpMatrix, type3: FormatSpec) -> np.ndarray:
    """C = A @ B on the tensor cores (FP32 accumulation in TMEM).  Defined
    exactly where the reference's per-step type3-rounded result is the exact
    product (always true for slice operands, the pipeline's only use); other
    operands raise NotImplementedError instead of returning a differently
    rounded result."""
    if A.shape[1] != B.shape[0]:
        raise ValueError("inner dimensions do not match")
    if 2 * max(A.fmt.mant_bits, B.fmt.mant_bits) > 53:
        raise AssertionError("operand products would not be exact in FP64")
    if A.fmt.name != B.fmt.name:
        raise NotImplementedError("mixed operand formats are not wired to tcgen05 in this build")
    if type3.mant_bits > 24:
        raise NotImplementedError("accumulators wider than FP32 are not available on the tensor cores")
    if not accumulation_is_exact(A.data, B.data, type3):
        raise NotImplementedError(
            f"lp_gemm: this product's {type3.name} accumulation can round; the tensor-core path computes "
            "exact products only (per-step type3 rounding, lpgemm.py:49-77, is not implemented)")
    torch = _lib.require_cuda()
    m, k = A.shape
    n = B.shape[1]
    if k == 0 or m == 0 or n == 0:
        return np.zeros((m, n))
    ca = encode_values(A.data, A.fmt)
    cb = encode_values(np.ascontiguousarray(B.data.T), B.fmt)  # K-major B
    fp6 = A.fmt.name in ("fp6e3m2", "fp6e2m3")
    ta, lda = _padded_codes(torch, ca, fp6)
    tb, ldb = _padded_codes(torch, cb, fp6)
    D = torch.empty((m, n), dtype=torch.float32, device="cuda")
    _lib.call("oz_lp_gemm", ta.data_ptr(), tb.data_ptr(), lda, ldb, m, n, k, _lib.FMT_CODE[A.fmt.name],
              D.data_ptr(), n, _lib.stream_ptr(torch))
    out = D.double().cpu().numpy()
    if not np.all(np.isfinite(out)):
        raise OverflowError("accumulation overflowed fp32")
    return out
