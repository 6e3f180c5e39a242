"""Error-free slicing of FP64 matrices along the inner dimension — B200 backend.

Host-side planning mirrors ``ozdgemm.slicing`` (slicing.py:45-97): the same
``SlicingParams`` / ``compute_params`` / ``predict_*`` contract.  The slicing
itself (slicing.py:128-206) runs on the GPU in ``oz_split.cu``:

  1. one fused pass (``oz_split_fused``): FP8/FP16 code planes, K-major
     ``[s][rows][ld]``, int32 exponents ``[s][rows]``, per-row slice counts,
     the global slice count s and the validation flags;
  2. ``oz_split_pad`` zero-fills the planes of rows that ended before s.
  (Exact two-pass fallback, ``oz_split_count`` + ``oz_split_rows``, when a
  row needs more planes than were allocated.)

Columns of B are sliced by transposing B on the device first (the reference
does the same transpose on the host, slicing.py:199-203).  ``slice_matrix``
returns a reference-compatible ``SliceSet`` (float64 coefficient planes and
integer exponents) decoded from the device planes; ``oz_gemm`` keeps the
device planes (``DeviceSlices``) and never decodes them.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import SlicingInfeasible
from .formats import FormatSpec, decode_codes

__all__ = [
    "SlicingInfeasible", "SlicingParams", "SliceSet", "DeviceSlices", "compute_params",
    "predict_slice_count", "predict_gemm_count", "slice_vector", "slice_matrix", "split_rows_device",
    "split_many_device", "split_deferred",
]


@dataclass(frozen=True)
class SlicingParams:
    """Slicing constants for significand widths m1 (input), m2 (slice storage),
    m3 (accumulator) at inner dimension k (slicing.py:45-69)."""

    m1: int
    m2: int
    m3: int
    k: int
    gamma: int
    xi: int
    rho: int
    slice_width: int = field(init=False)

    def __post_init__(self):
        object.__setattr__(self, "slice_width", self.m1 - self.rho)

    @property
    def feasible(self) -> bool:
        return self.slice_width >= 0


def compute_params(m1: int, m2: int, m3: int, k: int) -> SlicingParams:
    """gamma = ceil(m1 - (m3 - log2 k)/2), xi = m1 - m2, rho = max(gamma, xi)
    (slicing.py:72-81; paper Eqs. for the error-free accumulation bound)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    if min(m1, m2, m3) < 1:
        raise ValueError("significand bit counts must be >= 1")
    gamma = math.ceil(m1 - (m3 - math.log2(k)) / 2)
    xi = m1 - m2
    return SlicingParams(m1, m2, m3, k, gamma, xi, max(gamma, xi))


def predict_slice_count(params: SlicingParams):
    """Slices for a fully filled m1-bit significand (slicing.py:84-88), or None."""
    if not params.feasible:
        return None
    return -(-params.m1 // (params.slice_width + 1))


def predict_gemm_count(m1: int, m2: int, m3: int, k: int):
    """Square of the predicted slice count (slicing.py:91-97), or None."""
    s = predict_slice_count(compute_params(m1, m2, m3, k))
    return None if s is None else s * s


@dataclass
class SliceSet:
    """Reference-compatible slices (slicing.py:100-116): ``coeff[p]`` has the
    input's shape with exact float64 coefficient values, ``expo[p]`` one int per
    row ("rows") or column ("cols")."""

    orientation: str
    s: int
    coeff: list
    expo: list
    params: SlicingParams
    fmt: FormatSpec


@dataclass
class DeviceSlices:
    """Slices resident in HBM, laid out for TMA: ``planes`` uint8
    ``[s, rows, ld * elem_bytes]`` (K-major codes, zero padded), ``expo`` int32
    ``[s, rows]``, ``row_cnt`` int32 ``[rows]`` (per-row slice counts).
    Deferred splits (no host sync) hold ``cap`` planes, ``s`` = cap, and the
    true s and the flag word in the device tensor ``sf`` = [s, flags]."""

    planes: object
    expo: object
    row_cnt: object
    s: int
    rows: int
    kb: int
    ld: int
    fmt: FormatSpec
    sf: object = None
    host_flags: int = 0  # split_many_device: this matrix's flag word (read at its sync)

    def codes(self):
        """Codes as a [s, rows, kb] uint8/uint16 torch tensor view."""
        import torch

        if self.fmt.name in ("fp6e3m2", "fp6e2m3"):
            return torch.from_numpy(unpack_fp6(self.planes.cpu().numpy())[:, :, : self.kb])
        v = self.planes if _lib.ELEM_BYTES[self.fmt.name] == 1 else self.planes.view(torch.int16)
        return v[:, :, : self.kb]


def _row_bytes(ld: int, fmt: FormatSpec) -> int:
    """Bytes of one plane row of ld codes (packed FP6: 6 bits per code)."""
    if fmt.name in ("fp6e3m2", "fp6e2m3"):
        return ld * 3 // 4
    return ld * _lib.ELEM_BYTES[fmt.name]


def _row_len(kb: int, fmt: FormatSpec) -> int:
    """Elements per plane row: a multiple of 16 bytes, or of 128 codes for the
    packed FP6 layout (16 six-bit codes per 16-byte group, TMA 16U6_ALIGN16B)."""
    if fmt.name in ("fp6e3m2", "fp6e2m3"):
        return -(-kb // 128) * 128
    eb = _lib.ELEM_BYTES[fmt.name]
    return -(-kb // (16 // eb)) * (16 // eb)


def unpack_fp6(packed: np.ndarray) -> np.ndarray:
    """[..., ld*3/4] densely packed bytes (12 bytes of little-endian 6-bit codes
    per 16 codes) -> [..., ld] uint8 codes."""
    g = packed.reshape(*packed.shape[:-1], -1, 12).astype(np.uint64)
    lo = g[..., 0] | (g[..., 1] << 8) | (g[..., 2] << 16) | (g[..., 3] << 24) | (g[..., 4] << 32) | \
        (g[..., 5] << 40) | (g[..., 6] << 48) | (g[..., 7] << 56)
    hi = g[..., 8] | (g[..., 9] << 8) | (g[..., 10] << 16) | (g[..., 11] << 24)
    out = np.empty(g.shape[:-1] + (16,), dtype=np.uint8)
    for j in range(16):
        b = 6 * j
        if b + 6 <= 64:
            v = (lo >> np.uint64(b)) & np.uint64(63)
        elif b >= 64:
            v = (hi >> np.uint64(b - 64)) & np.uint64(63)
        else:
            v = ((lo >> np.uint64(b)) | (hi << np.uint64(64 - b))) & np.uint64(63)
        out[..., j] = v.astype(np.uint8)
    return out.reshape(*packed.shape[:-1], packed.shape[-1] // 3 * 4)


def _fmt_code(fmt: FormatSpec) -> int:
    if fmt.name not in _lib.FMT_CODE:
        raise NotImplementedError(
            f"slice format {fmt.name!r} has no tensor-core path on sm_100a in this build "
            f"(supported: {', '.join(_lib.FMT_CODE)})")
    return _lib.FMT_CODE[fmt.name]


def split_rows_device(X, fmt: FormatSpec, params: SlicingParams, emu: bool, stream=None,
                      check: bool = True) -> tuple[DeviceSlices, int]:
    """Slice every row of the CUDA float64 matrix view X (rows x kb, unit
    column stride) on the GPU.  Returns (slices, flags); raises the reference's
    exceptions when ``check``."""
    (ds,), flags = split_many_device([X], fmt, params, emu, stream, check)
    return ds, flags


PLANE_CAP = int(os.environ.get("OZ_PLANE_CAP", "32"))
PLANE_BUDGET_BYTES = 24 << 30  # per operand; larger operands start with fewer planes


def _plane_cap(rows: int, row_bytes: int, predicted: int) -> int:
    per_plane = max(rows * row_bytes, 1)
    cap = min(PLANE_CAP, max(PLANE_BUDGET_BYTES // per_plane, 1))
    return max(cap, min(predicted + 4, PLANE_CAP), 1)


def _is_col_view(X) -> bool:
    """X is the transpose view of a row-major matrix (its rows are columns):
    sliced in place by oz_split_fixed_cols (fixed-step mode with a plane limit)."""
    return X.shape[1] > 1 and X.stride(1) != 1 and (X.stride(0) == 1 or X.shape[0] == 1)


def _check_view(X, fixed: bool, max_planes: int):
    torch = _lib.require_cuda()
    if X.dtype != torch.float64:
        raise ValueError("split expects a float64 view")
    if X.stride(1) != 1 and X.shape[1] > 1 and not (fixed and max_planes > 0 and _is_col_view(X)):
        raise ValueError("split expects a float64 view with unit column stride (or, fixed-step mode with a "
                         "plane limit, the transpose view of a row-major matrix)")


def _split_launch(fixed: bool, max_planes: int, X, rows, kb, ldx, code, rho, emu, cap, planes, ld, expo, row_cnt,
                  s_ptr, f_ptr, sp):
    """oz_split_fused (reference exponents) or oz_split_fixed (fixed-step extension);
    a transpose view X = M[lo:hi, j0:j1].t() in fixed mode with a plane limit is
    sliced column by column in place (oz_split_fixed_cols, no transposed copy).
    The scratch tensor is allocated on, and used by, torch's current stream."""
    if fixed and max_planes > 0 and _is_col_view(X):
        torch = _lib.require_cuda()
        scratch = torch.empty(max(3 * rows, 1), dtype=torch.int32, device=X.device)
        _lib.call("oz_split_fixed_cols", X.data_ptr(), kb, rows, X.stride(1), code, rho, int(emu), cap, max_planes,
                  planes, ld, expo, row_cnt.data_ptr(), s_ptr, f_ptr, scratch.data_ptr(), sp)
        return
    if fixed:
        _lib.call("oz_split_fixed", X.data_ptr(), rows, kb, ldx, code, rho, int(emu), cap, max_planes, planes, ld,
                  expo, row_cnt.data_ptr(), s_ptr, f_ptr, sp)
    else:
        _lib.call("oz_split_fused", X.data_ptr(), rows, kb, ldx, code, rho, int(emu), cap, planes, ld, expo,
                  row_cnt.data_ptr(), s_ptr, f_ptr, sp)


def split_many_device(Xs, fmt: FormatSpec, params: SlicingParams, emu: bool, stream=None,
                      check: bool = True, flags_out=None, fixed: bool = False, max_planes: int = 0):
    """Slice several matrices with one host synchronisation.

    Fast path: one fused pass per matrix (``oz_split_fused``) writes the slices
    into a buffer of ``cap`` planes while counting; after the single sync that
    reads every s and flag word, ``oz_split_pad`` zero-fills the planes of rows
    that ended early.  A matrix with a row needing more than ``cap`` planes is
    re-sliced exactly with the two-pass path (count, then write s planes).
    Flags are checked in argument order (the reference slices A before B).
    Representability flags go to the device word ``flags_out`` if given
    (checked later by the caller), else they are checked here.  ``fixed``:
    fixed-step exponents (oz_split_fixed, opt-in extension), at most
    ``max_planes`` slices per row when > 0."""
    torch = _lib.require_cuda()
    if not params.feasible:
        raise SlicingInfeasible(
            f"slice width {params.slice_width} < 0 for m2={params.m2}, m3={params.m3}, k={params.k}")
    code = _fmt_code(fmt)
    sp = stream if stream is not None else _lib.stream_ptr(torch)
    eb = _lib.ELEM_BYTES[fmt.name]
    predicted = predict_slice_count(params) or 1
    metas = []
    small = torch.zeros(2 * len(Xs), dtype=torch.int32, device=Xs[0].device)  # [s, flags] per matrix
    for i, X in enumerate(Xs):
        rows, kb = X.shape
        _check_view(X, fixed, max_planes)
        ldx = X.stride(0) if rows > 1 else kb
        ld = _row_len(kb, fmt)
        cap = _plane_cap(rows, _row_bytes(ld, fmt), predicted)
        if fixed and max_planes > 0:
            cap = min(cap, max_planes)
        row_cnt = torch.zeros(max(rows, 1), dtype=torch.int32, device=X.device)
        planes = torch.empty((cap, rows, _row_bytes(ld, fmt)), dtype=torch.uint8, device=X.device)
        expo = torch.empty((cap, rows), dtype=torch.int32, device=X.device)
        if rows > 0:
            _split_launch(fixed, max_planes, X, rows, kb, ldx, code, params.rho, emu, cap, planes.data_ptr(), ld,
                          expo.data_ptr(), row_cnt, small.data_ptr() + 8 * i, small.data_ptr() + 8 * i + 4, sp)
        metas.append((X, rows, kb, ldx, ld, row_cnt, planes, expo))
    host = small.cpu().tolist()  # the one synchronisation
    out, all_flags = [], 0
    for i, (X, rows, kb, ldx, ld, row_cnt, planes, expo) in enumerate(metas):
        s_max, flags = host[2 * i], host[2 * i + 1] & 0xFFFFFFFF
        if flags & _lib.FLAG_PLANE_CAP:
            # Some row needs more planes than allocated: exact two-pass split.
            del planes, expo
            cnt = torch.zeros(2, dtype=torch.int32, device=X.device)
            if fixed:  # count-only mode of the fixed-step split (no planes)
                _split_launch(True, max_planes, X, rows, kb, ldx, code, params.rho, emu, 0, None, ld, None,
                              row_cnt, cnt.data_ptr(), cnt.data_ptr() + 4, sp)
            else:
                _lib.call("oz_split_count", X.data_ptr(), rows, kb, ldx, code, params.rho, int(emu),
                          row_cnt.data_ptr(), cnt.data_ptr(), cnt.data_ptr() + 4, sp)
            s_max, flags = (int(v) for v in cnt.cpu().tolist())
            flags &= 0xFFFFFFFF
            if check:
                _lib.raise_for_flags(flags, "split")
            planes = torch.empty((s_max, rows, _row_bytes(ld, fmt)), dtype=torch.uint8, device=X.device)
            expo = torch.empty((s_max, rows), dtype=torch.int32, device=X.device)
            if s_max > 0:
                fw = torch.zeros(1, dtype=torch.int32, device=X.device)
                fwp = (flags_out if flags_out is not None else fw).data_ptr()
                if fixed:
                    s_scr = torch.zeros(1, dtype=torch.int32, device=X.device)
                    _split_launch(True, max_planes, X, rows, kb, ldx, code, params.rho, emu, s_max,
                                  planes.data_ptr(), ld, expo.data_ptr(), row_cnt, s_scr.data_ptr(), fwp, sp)
                    _lib.call("oz_split_pad", planes.data_ptr(), ld, rows, code, s_max, None, row_cnt.data_ptr(),
                              None, sp)
                else:
                    _lib.call("oz_split_rows", X.data_ptr(), rows, kb, ldx, code, params.rho, int(emu), s_max,
                              planes.data_ptr(), ld, expo.data_ptr(), row_cnt.data_ptr(), fwp, sp)
                if flags_out is None:
                    flags |= int(fw.item()) & 0xFFFFFFFF  # representability (write pass only)
                    if check:
                        _lib.raise_for_flags(flags, "split")
            full = flags
        else:
            full = flags
            rep = flags & _lib.FLAG_NOT_REPRESENTABLE
            flags &= ~_lib.FLAG_NOT_REPRESENTABLE
            if check:
                _lib.raise_for_flags(flags, "split")
            if rep:
                if flags_out is not None:
                    flags_out.bitwise_or_(rep)
                elif check:
                    _lib.raise_for_flags(rep, "split")
            planes, expo = planes[:s_max], expo[:s_max]
            if s_max > 0 and rows > 0:
                _lib.call("oz_split_pad", planes.data_ptr(), ld, rows, code, s_max,
                          None if fixed else expo.data_ptr(), row_cnt.data_ptr(), None, sp)
        all_flags |= flags
        out.append(DeviceSlices(planes, expo, row_cnt[:rows], s_max, rows, kb, ld, fmt, host_flags=full))
    return out, all_flags


class Arena:
    """Named flat device buffers reused across the passes of one panelled
    oz_gemm call (all on one stream, so a pass's reuse is ordered after the
    previous pass's GEMM): without it every panel allocates ~GiB-sized plane
    buffers while the previous ones are being freed, and near the memory limit
    the caching allocator falls back to synchronous cudaFree / cudaMalloc."""

    def __init__(self, torch, device):
        self.torch, self.device, self.bufs = torch, device, {}

    def take(self, name: str, shape, dtype):
        n = 1
        for d in shape:
            n *= int(d)
        nbytes = max(n * self.torch.empty((), dtype=dtype).element_size(), 1)
        buf = self.bufs.get(name)
        if buf is None or buf.numel() < nbytes:
            self.bufs.pop(name, None)
            buf = self.bufs[name] = self.torch.empty(nbytes, dtype=self.torch.uint8, device=self.device)
        return buf[:nbytes].view(dtype).view(*shape) if n else buf[:0].view(dtype).view(*shape)


def split_deferred(X, fmt: FormatSpec, params: SlicingParams, emu: bool, stream=None, fixed: bool = False,
                   max_planes: int = 0, arena: Arena | None = None, slot: str = "") -> DeviceSlices:
    """One-pass split without a host synchronisation: the fused split and the
    zero padding (which reads s on the device) are only enqueued.  The result
    holds ``cap`` planes; the pair GEMM takes the true s from ``sf`` on the
    device.  The caller reads ``sf`` later and must redo the work with
    ``split_many_device`` if its flags carry ``FLAG_PLANE_CAP``.  ``arena`` /
    ``slot``: take the planes, exponents and counts from reused buffers."""
    torch = _lib.require_cuda()
    code = _fmt_code(fmt)
    sp = stream if stream is not None else _lib.stream_ptr(torch)
    eb = _lib.ELEM_BYTES[fmt.name]
    rows, kb = X.shape
    _check_view(X, fixed, max_planes)
    ldx = X.stride(0) if rows > 1 else kb
    ld = _row_len(kb, fmt)
    cap = _plane_cap(rows, _row_bytes(ld, fmt), predict_slice_count(params) or 1)
    if fixed and max_planes > 0:
        cap = min(cap, max_planes)
    sf = torch.zeros(2, dtype=torch.int32, device=X.device)  # read at the end: never shared
    if arena is not None:
        row_cnt = arena.take(slot + "cnt", (max(rows, 1),), torch.int32)
        planes = arena.take(slot + "planes", (cap, rows, _row_bytes(ld, fmt)), torch.uint8)
        expo = arena.take(slot + "expo", (cap, rows), torch.int32)
    else:
        row_cnt = torch.empty(max(rows, 1), dtype=torch.int32, device=X.device)
        planes = torch.empty((cap, rows, _row_bytes(ld, fmt)), dtype=torch.uint8, device=X.device)
        expo = torch.empty((cap, rows), dtype=torch.int32, device=X.device)
    if rows > 0:
        _split_launch(fixed, max_planes, X, rows, kb, ldx, code, params.rho, emu, cap, planes.data_ptr(), ld,
                      expo.data_ptr(), row_cnt, sf.data_ptr(), sf.data_ptr() + 4, sp)
        _lib.call("oz_split_pad", planes.data_ptr(), ld, rows, code, cap, None if fixed else expo.data_ptr(),
                  row_cnt.data_ptr(), sf.data_ptr(), sp)
    return DeviceSlices(planes, expo, row_cnt[:rows], cap, rows, kb, ld, fmt, sf)


def _to_device_f64(M):
    torch = _lib.require_cuda()
    if isinstance(M, torch.Tensor):
        t = M.to(device="cuda", dtype=torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(M, dtype=np.float64))).to("cuda")
    return t.contiguous()


def transpose_device(X, arena: Arena | None = None):
    """Device transpose (kernel ``oz_transpose``) of a 2-D float64 CUDA tensor."""
    torch = _lib.require_cuda()
    rows, cols = X.shape
    if X.stride(1) != 1:
        X = X.contiguous()
    out = arena.take("Bt", (cols, rows), torch.float64) if arena is not None else \
        torch.empty((cols, rows), dtype=torch.float64, device=X.device)
    if rows and cols:
        _lib.call("oz_transpose", X.data_ptr(), rows, cols, X.stride(0) if rows > 1 else cols,
                  out.data_ptr(), rows, _lib.stream_ptr(torch))
    return out


def slice_matrix(M, orientation: str, fmt: FormatSpec, params: SlicingParams,
                 arith: str = "fp64") -> SliceSet:
    """GPU replacement of ``ozdgemm.slice_matrix`` (slicing.py:190-206).

    "rows" slices each row (left operand); "cols" each column (right operand).
    ``arith`` selects hardware FP64 ("fp64") or the integer-only emulation
    ("emu") inside the split kernel; both give identical bits."""
    torch = _lib.require_cuda()
    is_torch = isinstance(M, torch.Tensor)
    if not is_torch:
        M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2:
        raise ValueError("slice_matrix expects a 2-D matrix")
    if orientation not in ("rows", "cols"):
        raise ValueError("orientation must be 'rows' or 'cols'")
    if arith not in ("fp64", "emu"):
        raise ValueError("arith must be 'fp64' or 'emu'")
    X = _to_device_f64(M)
    if orientation == "cols":
        X = transpose_device(X)
    ds, _ = split_rows_device(X, fmt, params, arith == "emu")
    return device_to_sliceset(ds, orientation, params, as_torch=is_torch)


def device_to_sliceset(ds: DeviceSlices, orientation: str, params: SlicingParams,
                       as_torch: bool = False) -> SliceSet:
    """Decode device planes into the reference's SliceSet representation."""
    torch = _lib.require_cuda()
    codes = ds.codes().cpu().numpy()
    vals = decode_codes(codes if codes.dtype == np.uint8 else codes.view(np.uint16), ds.fmt.name)
    expo = ds.expo.cpu().numpy().astype(np.int64)
    coeff = [vals[p] if orientation == "rows" else np.ascontiguousarray(vals[p].T) for p in range(ds.s)]
    expos = [expo[p] for p in range(ds.s)]
    if as_torch:
        coeff = [torch.from_numpy(c).cuda() for c in coeff]
        expos = [torch.from_numpy(e).cuda() for e in expos]
    return SliceSet(orientation, ds.s, coeff, expos, params, ds.fmt)


def slice_vector(x, fmt: FormatSpec, params: SlicingParams, arith: str = "fp64"):
    """Slice one length-k vector (slicing.py:180-187)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 1:
        raise ValueError("slice_vector expects a 1-D vector")
    ss = slice_matrix(x[None, :], "rows", fmt, params, arith)
    return [c[0] for c in ss.coeff], [int(e[0]) for e in ss.expo]
