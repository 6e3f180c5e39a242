"""CPU oracle for the Ozaki-scheme DGEMM hot path — TEST INFRASTRUCTURE ONLY.

A ctypes front end to ``oz_oracle.c``, the C restatement of the reference
``ozdgemm`` 1.0.0 algorithm (see the citations in that file).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may
import this package, and only as the checker / the timed CPU reference — the
product package never touches it.

Pinned against golden vectors produced by the reference itself
(``tests/golden/gen_golden.py``; checked in ``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import ctypes
import math
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB = _HERE / "liboz_oracle.so"
_lib = None

FMT_MANT = {"fp64": 53, "fp32": 24, "fp16": 11, "bf16": 8, "fp8e4m3": 4, "fp8e5m2": 3,
            "fp6e3m2": 3, "fp6e2m3": 4}


def build() -> Path:
    """Compile oz_oracle.c with the committed Makefile (gcc, no reference sources)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = ctypes.CDLL(str(LIB))
        P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        lib.oro_split_rows.restype = I
        lib.oro_split_rows.argtypes = [P, I64, I64, I64, I, I, I, P, P, P, P]
        lib.oro_pair_block.restype = None
        lib.oro_pair_block.argtypes = [P, P, P, P, I64, I64, I64, I, I, I, I, I, I, I, P, I, P]
        lib.oro_emu_add.restype = ctypes.c_uint64
        lib.oro_emu_add.argtypes = [ctypes.c_uint64, ctypes.c_uint64, P]
        lib.oro_max_threads.restype = I
        lib.oro_dd_gemm.restype = None
        lib.oro_dd_gemm.argtypes = [P, P, P, I64, I64, I64, I]
        _lib = lib
    return _lib


def max_threads() -> int:
    return _load().oro_max_threads()


def compute_rho(m1: int, m2: int, m3: int, k: int) -> tuple[int, bool]:
    """(rho, feasible) — restates slicing.compute_params (slicing.py:72-81)."""
    gamma = math.ceil(m1 - (m3 - math.log2(k)) / 2)
    rho = max(gamma, m1 - m2)
    return rho, (m1 - rho) >= 0


def emu_add(a: float, b: float) -> tuple[float, int]:
    flags = ctypes.c_uint32(0)
    ab = np.array([a], dtype=np.float64).view(np.uint64)[0]
    bb = np.array([b], dtype=np.float64).view(np.uint64)[0]
    r = _load().oro_emu_add(int(ab), int(bb), ctypes.byref(flags))
    return float(np.array([r], dtype=np.uint64).view(np.float64)[0]), flags.value


def split_rows(X, rho: int, emu: bool = False, cap: int = 64):
    """Slice each row of X.  Returns (coeff [s, rows, kb] float64,
    expo [s, rows] int32, row counts [rows], s, flags)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    rows, kb = X.shape
    lib = _load()
    while True:
        coeff = np.zeros((cap, rows, kb), dtype=np.float64)
        expo = np.zeros((cap, rows), dtype=np.int32)
        cnt = np.zeros(rows, dtype=np.int32)
        flags = ctypes.c_uint32(0)
        s = lib.oro_split_rows(X.ctypes.data, rows, kb, kb, rho, int(emu), cap, coeff.ctypes.data,
                               expo.ctypes.data, cnt.ctypes.data, ctypes.byref(flags))
        if s >= 0:
            return coeff[:s].copy(), expo[:s].copy(), cnt, s, flags.value
        cap *= 2


def slice_matrix(M, orientation: str, rho: int, emu: bool = False):
    """(coeff list, expo list, s, flags) in the reference's SliceSet convention."""
    M = np.asarray(M, dtype=np.float64)
    X = M if orientation == "rows" else np.ascontiguousarray(M.T)
    coeff, expo, _, s, flags = split_rows(X, rho, emu)
    if orientation == "cols":
        coeff = [np.ascontiguousarray(c.T) for c in coeff]
    return list(coeff), [e.astype(np.int64) for e in expo], s, flags


def oz_gemm(A, B, type2: str = "fp8e4m3", type3: str = "fp32", k_block: int = 0, emu: bool = False,
            max_slices=None, order: str = "smallest-first", pair_cutoff=None, nthreads: int | None = None):
    """Full reference pipeline on the CPU.  Returns (C, info) with
    info = {"blocks": [(lo, hi, sx, sy)], "flags": int}."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    m, k = A.shape
    n = B.shape[1]
    lib = _load()
    nthreads = nthreads or max_threads()
    m2, m3 = FMT_MANT[type2], FMT_MANT[type3]
    C = np.zeros((m, n), dtype=np.float64)
    blocks = [(0, k)] if k_block == 0 else [(lo, min(lo + k_block, k)) for lo in range(0, k, k_block)]
    info = {"blocks": [], "flags": 0}
    for bi, (lo, hi) in enumerate(blocks):
        kb = hi - lo
        rho, feasible = compute_rho(53, m2, m3, kb)
        if not feasible:
            raise ValueError("infeasible slicing parameters")
        ca, ea, _, sa, fa = split_rows(A[:, lo:hi], rho, emu)
        cbt, eb, _, sb, fb = split_rows(np.ascontiguousarray(B[lo:hi, :].T), rho, emu)
        info["flags"] |= fa | fb
        if fa | fb:
            return C, info
        cb = np.ascontiguousarray(cbt.transpose(0, 2, 1))  # [s][kb][n]
        sx = min(sa, max_slices or sa)
        sy = min(sb, max_slices or sb)
        info["blocks"].append((lo, hi, sx, sy))
        flags = ctypes.c_uint32(0)
        fp32 = 1 if type3 == "fp32" else 0
        if sx and sy:
            lib.oro_pair_block(np.ascontiguousarray(ca).ctypes.data, np.ascontiguousarray(ea).ctypes.data,
                               cb.ctypes.data, np.ascontiguousarray(eb).ctypes.data, m, n, kb, sx, sy,
                               0 if order == "smallest-first" else 1,
                               -1 if pair_cutoff is None else pair_cutoff, int(emu), fp32, int(bi > 0),
                               C.ctypes.data, nthreads, ctypes.byref(flags))
        elif bi == 0:
            C[:] = 0.0
        info["flags"] |= flags.value
    return C, info


def dd_gemm(A, B, nthreads: int | None = None):
    """Double-double GEMM with one final rounding (accuracy checker for the
    acceptance criteria; pinned to the reference's exact ref_gemm by tests)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    m, k = A.shape
    n = B.shape[1]
    C = np.empty((m, n), dtype=np.float64)
    _load().oro_dd_gemm(A.ctypes.data, B.ctypes.data, C.ctypes.data, m, n, k, nthreads or max_threads())
    return C


def naive_gemm(A, B):
    """Triple-loop FP64 GEMM, ascending-k sequential accumulation (restates
    oracle.naive_gemm_fp64, oracle.py:177-188)."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    C = np.zeros((A.shape[0], B.shape[1]))
    for t in range(A.shape[1]):
        C += A[:, t, None] * B[t, None, :]
    return C
