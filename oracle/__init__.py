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


def split_rows_fixed(X, rho: int, max_planes: int = 0):
    """Fixed-step slicing (the opt-in ``slice_exponents="fixed"`` extension; no
    reference counterpart): the reference's _slice_rows iteration
    (slicing.py:144-176) with c_p = c_0 - p (54 - rho), c_0 = ceil_log2 max|x|.
    Returns (coeff [s, rows, kb], expo [s, rows], counts, s)."""
    X = np.array(X, dtype=np.float64)
    rows, kb = X.shape
    w = 54 - rho
    mx = np.max(np.abs(X), axis=1) if kb else np.zeros(rows)
    m, e = np.frexp(np.where(mx > 0, mx, 1.0))
    c0 = np.where(mx > 0, np.where(m == 0.5, e - 1, e), 0).astype(np.int64)
    coeffs, cnt, p = [], np.zeros(rows, dtype=np.int64), 0
    while np.any(X != 0) and (max_planes <= 0 or p < max_planes):
        active = np.any(X != 0, axis=1)
        c = c0 - p * w
        sigma = np.ldexp(1.5, c + rho - 1)[:, None]
        v = (X + sigma) - sigma
        v[~active] = 0.0
        X = X - v
        coeffs.append(np.ldexp(v, -c[:, None]))
        cnt[active] = p + 1
        p += 1
    s = len(coeffs)
    expo = np.stack([c0 - q * w for q in range(s)]) if s else np.zeros((0, rows), dtype=np.int64)
    coeff = np.stack(coeffs) if s else np.zeros((0, rows, kb))
    return coeff, expo, cnt, s


def oz_gemm_fixed(A, B, type2: str = "fp8e4m3", type3: str = "fp32", k_block: int = 0, max_slices=None,
                  order: str = "smallest-first", pair_cutoff=None, pad_to=None):
    """CPU restatement of the fixed-step, level-grouped pipeline
    (GemmConfig.slice_exponents="fixed"): per block, pairs in the reference order
    (ozgemm.py:179-183, restricted to p+q <= pair_cutoff), consecutive pairs of one
    anti-diagonal summed exactly in groups of at most group_max, each group added
    to Cb once as G * 2^(cA_p0 + cB_q0) with one RNE rounding, then C += Cb.
    ``pad_to`` = [(s_A, s_B)] per block: extend the slices with zero planes
    (continuing exponents) to those counts — a row/column sample of a larger
    problem then walks the same pair groups as the full problem.
    Returns (C, blocks [(lo, hi, sx, sy)])."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    m, k = A.shape
    n = B.shape[1]
    m2, m3 = FMT_MANT[type2], FMT_MANT[type3]
    blocks = [(0, k)] if k_block == 0 else [(lo, min(lo + k_block, k)) for lo in range(0, k, k_block)]
    C = np.zeros((m, n))
    info = []
    for bi, (lo, hi) in enumerate(blocks):
        kb = hi - lo
        rho, _ = compute_rho(53, m2, m3, kb)
        lim = [v for v in (max_slices, None if pair_cutoff is None else pair_cutoff + 1) if v]
        mp = min(lim) if lim else 0
        ca, ea, _, sa = split_rows_fixed(A[:, lo:hi], rho, mp)
        cbt, eb, _, sb = split_rows_fixed(B[lo:hi, :].T, rho, mp)
        if pad_to is not None:
            w = 54 - rho

            def pad(c, e, s, want):
                if want <= s:
                    return c, e, s
                c = np.concatenate([c, np.zeros((want - s,) + c.shape[1:])])
                e0 = e[0] if s else np.zeros(c.shape[1], dtype=np.int64)
                return c, np.stack([e0 - q * w for q in range(want)]), want

            ca, ea, sa = pad(ca, ea, sa, pad_to[bi][0])
            cbt, eb, sb = pad(cbt, eb, sb, pad_to[bi][1])
        sx, sy = min(sa, max_slices or sa), min(sb, max_slices or sb)
        info.append((lo, hi, sx, sy))
        gmax = max(1, min(64, (1 << (24 - 2 * (53 - rho))) // kb))
        pairs = [(p, q) for p in range(sx) for q in range(sy) if pair_cutoff is None or p + q <= pair_cutoff]
        sgn = -1 if order == "smallest-first" else 1
        pairs.sort(key=lambda pq: (sgn * (pq[0] + pq[1]), pq[0], pq[1]))
        Cb = np.zeros((m, n))
        i = 0
        while i < len(pairs):
            p0, q0 = pairs[i]
            G = np.zeros((m, n))
            j = i
            while j < len(pairs) and j - i < gmax and sum(pairs[j]) == p0 + q0:
                G += ca[pairs[j][0]] @ cbt[pairs[j][1]].T  # exact: small multiples of the slice grid
                j += 1
            Cb = Cb + np.ldexp(G, ea[p0][:, None] + eb[q0][None, :])
            i = j
        C = Cb.copy() if bi == 0 else C + Cb
    return C, info
