"""Inputs for the failure-semantics cases (shared by gen_golden.py, which records
what the REFERENCE raises or returns for each, and tests/test_gpu_errors.py,
which drives them through the CUDA path).  No reference import here.

Each case: name -> (A, B, config kwargs).  Config kwargs use format names:
{"type2": ..., "type3": ..., "k_block": ..., "fp64_emulation": ...}.
Covers slicing.py:119-125 (non-finite / subnormal input), slicing.py:155-158
(sigma out of range), ozgemm.py:132-140 and fp64emu.py:269-277 (scaled term out
of range, HW and emulated), ozgemm.py:147-154 (shapes, k_block), and the order
in which the reference raises (A's split, B's split, then the block's terms,
block by block).
"""

from __future__ import annotations

import numpy as np


def _r(seed, shape, lo=1.0, hi=2.0):
    rng = np.random.default_rng(seed)
    return lo + (hi - lo) * rng.random(shape)


def cases():
    f8 = {"type2": "fp8e4m3", "type3": "fp32"}
    out = {}
    # validation (slicing.py:119-125) and shapes (ozgemm.py:147-154)
    out["nan_input"] = (np.array([[1.0, np.nan]]), np.ones((2, 1)), f8)
    out["inf_input_B"] = (np.ones((1, 2)), np.array([[1.0], [np.inf]]), f8)
    out["subnormal_input"] = (np.array([[1.0, 5e-324]]), np.ones((2, 1)), f8)
    out["shape_mismatch"] = (np.ones((2, 3)), np.ones((2, 3)), f8)
    out["kblock_gt_k"] = (np.ones((2, 3)), np.ones((3, 2)), dict(f8, k_block=4))
    # the reference slices A before B: A's error wins
    out["order_A_nan_B_subnormal"] = (np.array([[1.0, np.nan]]), np.array([[1.0], [5e-324]]), f8)
    out["order_A_subnormal_B_nan"] = (np.array([[1.0, 5e-324]]), np.array([[1.0], [np.nan]]), f8)
    # sigma = 1.5 * 2^(c + rho - 1) beyond the largest binade (slicing.py:155-158)
    A = _r(1, (4, 8))
    A[2, 5] = 2.0 ** 990
    out["sigma_range"] = (A, _r(2, (8, 3)), f8)
    # scaled terms below the normal range: RangeError in both modes
    for fmt in ("fp8e4m3", "fp16", "bf16"):
        for emu in (False, True):
            cfg = {"type2": fmt, "type3": "fp32", "fp64_emulation": emu}
            out[f"term_subnormal_{fmt}_{'emu' if emu else 'hw'}"] = (
                _r(3, (5, 40)) * 2.0 ** -520, _r(4, (40, 6)) * 2.0 ** -520, cfg)
            # overflow: terms beyond 2^1024
            out[f"term_overflow_{fmt}_{'emu' if emu else 'hw'}"] = (
                _r(5, (5, 40)) * 2.0 ** 600, _r(6, (40, 6)) * 2.0 ** 500, cfg)
    # HW mode: terms that underflow all the way round to +0 are accepted
    # (np.ldexp gives 0, ozgemm.py:136-139); the emulated scale2 raises instead.
    A = _r(7, (4, 16))
    A[0] *= 2.0 ** -600  # row 0: every term below 2^-1090 (B ~ 2^-500)
    for emu in (False, True):
        out[f"term_to_zero_{'emu' if emu else 'hw'}"] = (A, _r(8, (16, 5)) * 2.0 ** -500,
                                                          {"type2": "fp8e4m3", "type3": "fp32",
                                                           "fp64_emulation": emu})
    # One slice per operand, G = 2^-20 by cancellation (FP16 grid 2^-11 at k = 3):
    # the term 2^-1028 is subnormal although G * 2^(eA+eB) with |G| >= 2^-8 would
    # be normal — guards the epilogue's exponent bounds for FP16/BF16 slices.
    A = np.array([[2.0 ** -514, 2.0 ** -504, 2.0 ** -504]])
    B = np.array([[2.0 ** -514], [2.0 ** -504], [-(2.0 ** -504)]])
    for emu in (False, True):
        out[f"term_tiny_G_fp16_{'emu' if emu else 'hw'}"] = (A, B, {"type2": "fp16", "type3": "fp32",
                                                                      "fp64_emulation": emu})
    # block order: block 0's terms fail before block 1's split sees the NaN
    A = _r(9, (3, 8))
    A[:, :4] *= 2.0 ** -520
    A[1, 6] = np.nan
    B = _r(10, (8, 4))
    B[:4] *= 2.0 ** -520
    out["block_order_term_then_nan"] = (A, B, dict(f8, k_block=4))
    return out
