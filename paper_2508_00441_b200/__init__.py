"""paper_2508_00441_b200 — Ozaki-scheme DGEMM on NVIDIA B200 (sm_100a).

Drop-in for the hot path of the reference package ``ozdgemm`` 1.0.0
(arXiv 2508.00441, "DGEMM without FP64 Arithmetic"): the same public names for
the split -> slice-pair GEMM -> accumulate path (ozdgemm/__init__.py:13-62),
computed by hand-written tcgen05/TMA kernels in ``liboz_b200.so`` behind the C
ABI of ``include/oz_b200.h``.  There is no CPU fallback: without the built
library and a CUDA device the compute entry points raise
``BackendUnavailable``.

The reference CLI's subcommands (slices-table, gemm, accuracy, verify) run on
this backend via ``python -m paper_2508_00441_b200.cli`` (same report schema).
Out of scope (not on the hot path): the scalar FP64-emulation
API (F64Word, emu_*), cvt/is_representable and the exact rational oracle
(ref_gemm, exact_gemm, naive_gemm_fp64).
"""

__version__ = "0.1.0"

from ._lib import BackendUnavailable
from .errors import DimensionError, RangeError, RepresentabilityError, SlicingInfeasible
from .formats import FORMATS, FormatSpec, get_format
from .lpgemm import LpMatrix, lp_gemm
from .metrics import max_rel_error
from .ozgemm import GemmConfig, OzResult, OzStats, oz_gemm, oz_gemm_count, oz_gemm_device, transpose
from .slicing import (SliceSet, SlicingParams, compute_params, predict_gemm_count, predict_slice_count,
                      slice_matrix, slice_vector)

__all__ = [
    "__version__", "BackendUnavailable",
    "FORMATS", "FormatSpec", "get_format",
    "RangeError", "SlicingInfeasible", "DimensionError", "RepresentabilityError",
    "SlicingParams", "SliceSet", "compute_params", "predict_slice_count", "predict_gemm_count",
    "slice_vector", "slice_matrix",
    "LpMatrix", "lp_gemm",
    "GemmConfig", "OzResult", "OzStats", "oz_gemm", "oz_gemm_count", "oz_gemm_device", "transpose",
    "max_rel_error",
]
