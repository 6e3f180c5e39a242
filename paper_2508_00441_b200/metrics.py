"""Error metric with the reference's definition (oracle.py:191-201)."""

from __future__ import annotations

import numpy as np


def max_rel_error(C, Cref) -> float:
    """max_ij |C_ij - Cref_ij| / |Cref_ij| (FP64 differences)."""
    C = np.asarray(C, dtype=np.float64)
    Cref = np.asarray(Cref, dtype=np.float64)
    if C.shape != Cref.shape:
        raise ValueError("shape mismatch")
    if np.any(Cref == 0):
        raise ZeroDivisionError("reference entry is zero; relative error undefined")
    return float(np.max(np.abs(C - Cref) / np.abs(Cref)))
