"""ctypes binding of liboz_b200.so (C ABI in include/oz_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is no CPU fallback: if the library or a CUDA device is
missing, every product entry point raises :class:`BackendUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "liboz_b200.so"

# Status codes and device flag bits (include/oz_b200.h).
OZ_OK, OZ_EINVAL, OZ_EUNSUPPORTED, OZ_ECUDA, OZ_ETMAP, OZ_ESLICES = range(6)
FMT_CODE = {"fp8e4m3": 0, "fp8e5m2": 1, "fp16": 2, "bf16": 3, "fp6e3m2": 4, "fp6e2m3": 5}
ELEM_BYTES = {"fp8e4m3": 1, "fp8e5m2": 1, "fp16": 2, "bf16": 2, "fp6e3m2": 1, "fp6e2m3": 1}
# Slice formats whose products run on the tensor cores (fp6e2m3 slices are never
# representable: SlicingInfeasible, as in the reference).
TC_FORMATS = ("fp8e4m3", "fp8e5m2", "fp16", "bf16", "fp6e3m2")

FLAG_NONFINITE_INPUT = 1 << 0
FLAG_SUBNORMAL_INPUT = 1 << 1
FLAG_SIGMA_RANGE = 1 << 2
FLAG_SLICE_CAP = 1 << 3
FLAG_NOT_REPRESENTABLE = 1 << 4
FLAG_EMU_RANGE = 1 << 5
FLAG_TERM_RANGE = 1 << 6
FLAG_SUBNORMAL_RESID = 1 << 7
FLAG_PLANE_CAP = 1 << 8  # oz_split_fused only: re-run the exact two-pass split

# Every symbol include/oz_b200.h declares, with its ctypes signature.
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
SIGNATURES = {
    "oz_split_fused": (_I, [_P, _I64, _I64, _I64, _I, _I, _I, _I, _P, _I64, _P, _P, _P, _P, _P]),
    "oz_split_fixed": (_I, [_P, _I64, _I64, _I64, _I, _I, _I, _I, _I, _P, _I64, _P, _P, _P, _P, _P]),
    "oz_split_fixed_cols": (_I, [_P, _I64, _I64, _I64, _I, _I, _I, _I, _I, _P, _I64, _P, _P, _P, _P, _P, _P]),
    "oz_split_fixed_cols_scratch": (ctypes.c_int64, [_I64]),
    "oz_split_pad": (_I, [_P, _I64, _I64, _I, _I, _P, _P, _P, _P]),
    "oz_split_count": (_I, [_P, _I64, _I64, _I64, _I, _I, _I, _P, _P, _P, _P]),
    "oz_split_rows": (_I, [_P, _I64, _I64, _I64, _I, _I, _I, _I, _P, _I64, _P, _P, _P, _P]),
    "oz_transpose": (_I, [_P, _I64, _I64, _I64, _P, _I64, _P]),
    "oz_tile_counts": (_I, [_P, _I64, _P, _P]),
    "oz_pair_gemm": (_I, [_P, _P, _I64, _I64, _I, _I, _P, _P, _P, _P, _I64, _I64, _I64, _I, _I, _I,
                          _I, _I, _I, _I, _P, _I64, _P, _P, _I64, _I, _P, _I64, _P, _P, _P]),
    "oz_pair_gemm_grouped": (_I, [_P, _P, _I64, _I64, _I, _I, _P, _P, _I64, _I64, _I64, _I, _I, _I, _I, _I, _I, _I,
                                  _I, _P, _I64, _P, _P, _I64, _I, _P, _I64, _P, _P, _P]),
    "oz_pair_gemm_workspace": (ctypes.c_int64, [_I64, _I64, _I64, _I, _I, _I, _I]),
    "oz_set_pair_variant": (_I, [_I, _I, _I]),
    "oz_set_epilogue_warps": (_I, [_I]),
    "oz_set_pair_schedule": (_I, [_I]),
    "oz_pair_plan": (_I, [_I64, _I64, _I64, _I, _I, _I, _I, _I, _I, _I, _P, _P]),
    "oz_lp_gemm": (_I, [_P, _P, _I64, _I64, _I64, _I64, _I64, _I, _P, _I64, _P]),
    "oz_emu_add_batch": (_I, [_P, _P, _P, _I64, _I, _P, _P]),
    "oz_dd_gemm": (_I, [_P, _P, _P, _I64, _I64, _I64, _P]),
    "oz_strerror": (ctypes.c_char_p, [_I]),
    "oz_version": (ctypes.c_char_p, []),
}


class BackendUnavailable(RuntimeError):
    """liboz_b200.so or a CUDA device is missing (no CPU fallback exists)."""


class LibError(RuntimeError):
    """A C-ABI call returned a non-OK status."""


_lib = None


def load(path: os.PathLike | None = None) -> ctypes.CDLL:
    """Load the shared library once and attach the declared signatures."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise BackendUnavailable(
            f"{p} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Invoke a C-ABI entry point; raise LibError on a non-OK status."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != OZ_OK:
        msg = lib.oz_strerror(rc).decode()
        if rc == OZ_EUNSUPPORTED:
            raise NotImplementedError(f"{name}: {msg}")
        raise LibError(f"{name} failed: {msg} (status {rc})")


def require_cuda():
    """Return torch with a usable CUDA device, or raise BackendUnavailable."""
    import torch

    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device: the B200 backend has no CPU fallback")
    load()
    return torch


def set_pair_variant(cta_group: int = 0, tile_n: int = 0, raster_group: int = 0) -> None:
    """Force oz_pair_gemm's kernel variant (0 = automatic).  Results are bitwise
    identical in every variant; tests use this to cover all of them."""
    call("oz_set_pair_variant", cta_group, tile_n, raster_group)


def stream_ptr(torch) -> int:
    return torch.cuda.current_stream().cuda_stream


def raise_for_flags(flags: int, where: str) -> None:
    """Map device error bits to the reference's exception classes."""
    if not flags:
        return
    from .errors import RangeError, SlicingInfeasible

    if flags & FLAG_NONFINITE_INPUT:
        raise ValueError("slicing input must be finite")
    if flags & FLAG_SUBNORMAL_INPUT:
        raise RangeError("slicing input must be normal or zero")
    if flags & FLAG_SIGMA_RANGE:
        raise RangeError("shift constant outside normal range")
    if flags & FLAG_NOT_REPRESENTABLE:
        raise SlicingInfeasible(f"slice coefficients not representable ({where})")
    if flags & FLAG_SUBNORMAL_RESID:
        raise RangeError("operand is not a normal finite FP64 value (or zero)")
    if flags & FLAG_EMU_RANGE:
        raise RangeError("emulated add result outside normal range")
    if flags & FLAG_TERM_RANGE:
        raise RangeError("scaled term left the FP64 normal range")
    if flags & FLAG_SLICE_CAP:
        raise AssertionError("slicing failed to terminate")
    raise RuntimeError(f"unknown device flags {flags:#x} ({where})")
