"""Floating-point format descriptors (metadata only).

Mirrors the catalog of ``ozdgemm.formats`` (formats.py:36-109): the same
``FormatSpec`` fields and the same eight names, so a ``GemmConfig`` built for
the reference is accepted unchanged.  On B200 a slice format is not simulated:
E4M3/E5M2 slices are stored as real FP8 bytes and FP16/BF16 slices as real
16-bit halves that the tcgen05 tensor cores consume directly.  ``mant_bits``
(significand bits incl. the hidden bit) is what feeds the slicing constants.

``decode_codes`` turns stored slice codes back into exact float64 values (the
representation the reference keeps its slices in) for parity checks and for
``slice_matrix`` returning numpy.
"""

from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np

__all__ = [
    "FormatSpec", "FORMATS", "FP64", "FP32", "FP16", "BF16", "FP8_E4M3", "FP8_E5M2",
    "FP6_E3M2", "FP6_E2M3", "get_format", "mant_bits", "unit_roundoff",
    "TENSOR_CORE_SLICE_FORMATS", "decode_codes",
]


@dataclass(frozen=True)
class FormatSpec:
    """Binary floating-point format: ``mant_bits`` includes the hidden bit,
    normal values lie in [2**exp_min, max_finite]."""

    name: str
    exp_bits: int
    mant_bits: int
    exp_max: int
    exp_min: int
    max_finite: float
    finite_only: bool = False

    def __post_init__(self):
        if self.mant_bits < 1 or self.exp_bits < 2:
            raise ValueError("need mant_bits >= 1 and exp_bits >= 2")

    @property
    def unit_roundoff(self) -> float:
        return 2.0 ** -self.mant_bits

    @property
    def min_subnormal(self) -> float:
        return 2.0 ** (self.exp_min - self.mant_bits + 1)

    def __repr__(self):
        return f"FormatSpec({self.name!r})"


def _ieee_like(name: str, e: int, p: int) -> FormatSpec:
    bias = (1 << (e - 1)) - 1
    return FormatSpec(name, e, p, bias, 1 - bias, (2.0 - 2.0 ** (1 - p)) * 2.0 ** bias)


FP64 = _ieee_like("fp64", 11, 53)
FP32 = _ieee_like("fp32", 8, 24)
FP16 = _ieee_like("fp16", 5, 11)
BF16 = _ieee_like("bf16", 8, 8)
FP8_E5M2 = _ieee_like("fp8e5m2", 5, 3)
# OCP FP8/FP6 variants without inf (E4M3 keeps only S.1111.111 as NaN).
FP8_E4M3 = FormatSpec("fp8e4m3", 4, 4, 8, -6, 448.0, True)
FP6_E3M2 = FormatSpec("fp6e3m2", 3, 3, 4, -2, 28.0, True)
FP6_E2M3 = FormatSpec("fp6e2m3", 2, 4, 2, 0, 7.5, True)

FORMATS = {f.name: f for f in (FP16, BF16, FP8_E4M3, FP8_E5M2, FP6_E3M2, FP6_E2M3, FP32, FP64)}

# Slice formats the sm_100a tensor cores take directly in this build
# (kind::f8f6f4 for the FP8 pair, kind::f16 for the 16-bit pair).
TENSOR_CORE_SLICE_FORMATS = ("fp8e4m3", "fp8e5m2", "fp16", "bf16")


def get_format(name: str) -> FormatSpec:
    key = name.lower()
    if key not in FORMATS:
        raise ValueError(f"unknown format {name!r}; known: {', '.join(FORMATS)}")
    return FORMATS[key]


def mant_bits(fmt: FormatSpec) -> int:
    return fmt.mant_bits


def unit_roundoff(fmt: FormatSpec) -> float:
    return fmt.unit_roundoff


def _minifloat_table(ebits: int, mbits: int, bias: int) -> np.ndarray:
    """Value of every 8-bit code of a sign/exp/mantissa minifloat (no inf/nan use)."""
    codes = np.arange(256)
    sign = np.where(codes >> (ebits + mbits) & 1, -1.0, 1.0)
    field = (codes >> mbits) & ((1 << ebits) - 1)
    mant = codes & ((1 << mbits) - 1)
    mag = np.where(field == 0, mant * 2.0 ** (1 - bias - mbits),
                   (1.0 + mant / 2.0 ** mbits) * 2.0 ** (field.astype(np.float64) - bias))
    return sign * mag


_E4M3_LUT = _minifloat_table(4, 3, 7)
_E5M2_LUT = _minifloat_table(5, 2, 15)
_E3M2_LUT = _minifloat_table(3, 2, 3)[:64]
_E2M3_LUT = _minifloat_table(2, 3, 1)[:64]
FP6_SHIFT = 0  # FP6 codes are handled unpacked (slicing.unpack_fp6), one per byte


def decode_codes(codes: np.ndarray, fmt_name: str) -> np.ndarray:
    """Exact float64 values of stored slice codes (uint8 or uint16 arrays)."""
    if fmt_name == "fp8e4m3":
        return _E4M3_LUT[codes.astype(np.intp)]
    if fmt_name == "fp8e5m2":
        return _E5M2_LUT[codes.astype(np.intp)]
    if fmt_name in ("fp6e3m2", "fp6e2m3"):
        lut = _E3M2_LUT if fmt_name == "fp6e3m2" else _E2M3_LUT
        return lut[(codes.astype(np.intp) >> FP6_SHIFT) & 63]
    if fmt_name == "fp16":
        return codes.astype(np.uint16).view(np.float16).astype(np.float64)
    if fmt_name == "bf16":
        return (codes.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
    raise ValueError(f"no slice storage for {fmt_name}")
