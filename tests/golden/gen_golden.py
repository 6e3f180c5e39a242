"""Generate golden vectors by running the REFERENCE package itself.

Run here (the container that has /root/reference):
    python tests/golden/gen_golden.py
It imports ozdgemm 1.0.0 from /root/reference/pkg/src, runs its public API on
small seeded inputs and writes compact .npz/.json fixtures next to this file.
The fixtures travel with the repo; nothing at test time reads /root/reference.

Fixtures
  params.json      compute_params / predict_* KATs over (m2, m3, k) incl. the
                   acceptance GEMM-count table (tests/test_acceptance.py:27-38)
  slices.npz       slice_matrix outputs (coeff bits, exponents, s) for rows and
                   cols, E4M3/E5M2/FP16/BF16, HW and emulated arithmetic
  gemm.npz         oz_gemm C bits + per-block (s_x, s_y) for option sweeps
  errors.json      exception class raised for invalid inputs/configs
  emu_add.npz      fp64emu.add_arrays on edge operands
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import ozdgemm as R  # noqa: E402
from ozdgemm import fp64emu  # noqa: E402


def spread(rng, r, c, phi):
    return (rng.random((r, c)) - 0.5) * np.exp(phi * rng.standard_normal((r, c)))


def gen_params():
    out = {"kats": [], "table": []}
    for m2 in (3, 4, 8, 11):
        for m3 in (8, 11, 24):
            for k in (1, 2, 3, 16, 100, 1024, 1025, 4096, 8192, 65536, 262144):
                p = R.compute_params(53, m2, m3, k)
                out["kats"].append({"m2": m2, "m3": m3, "k": k, "gamma": p.gamma, "xi": p.xi, "rho": p.rho,
                                    "width": p.slice_width, "feasible": p.feasible,
                                    "pred_s": R.predict_slice_count(p),
                                    "pred_g": R.predict_gemm_count(53, m2, m3, k)})
    for t2 in R.FORMATS:
        for t3 in ("fp32", "fp16"):
            for k in [8 << i for i in range(16)]:
                out["table"].append({"type2": t2, "type3": t3, "k": k,
                                     "count": R.predict_gemm_count(53, R.FORMATS[t2].mant_bits,
                                                                  R.FORMATS[t3].mant_bits, k)})
    (HERE / "params.json").write_text(json.dumps(out, indent=0))


SLICE_CASES = [
    # name, rows, cols, phi, fmt, arith, orientation, seed
    ("e4m3_rows_hw", 9, 37, 0.5, "fp8e4m3", "fp64", "rows", 1),
    ("e4m3_rows_emu", 9, 37, 0.5, "fp8e4m3", "emu", "rows", 1),
    ("e4m3_rows_wide", 16, 200, 4.0, "fp8e4m3", "fp64", "rows", 2),
    ("e4m3_cols_hw", 150, 12, 1.0, "fp8e4m3", "fp64", "cols", 3),
    ("fp16_rows_hw", 11, 64, 2.0, "fp16", "fp64", "rows", 4),
    ("fp16_cols_emu", 64, 10, 2.0, "fp16", "emu", "cols", 5),
    ("bf16_rows_hw", 8, 50, 0.5, "bf16", "fp64", "rows", 6),
    ("e5m2_rows_hw", 8, 50, 0.5, "fp8e5m2", "fp64", "rows", 7),
]


def gen_slices():
    store = {}
    for name, r, c, phi, fmt, arith, orient, seed in SLICE_CASES:
        rng = np.random.default_rng(seed)
        M = spread(rng, r, c, phi)
        M[0, :] = 0.0  # an all-zero row/col
        if orient == "rows":
            M[1, 3] = 1.0 + 2.0 ** -40  # a long tail (SPEC.md:213-215 style)
        k = c if orient == "rows" else r
        f = R.get_format(fmt)
        params = R.compute_params(53, f.mant_bits, 24, k)
        ss = R.slice_matrix(M, orient, f, params, arith)
        store[f"{name}/M"] = M
        store[f"{name}/coeff"] = np.stack(ss.coeff).view(np.uint64)
        store[f"{name}/expo"] = np.stack(ss.expo).astype(np.int64)
        store[f"{name}/meta"] = np.array([ss.s, params.rho, k], dtype=np.int64)
    np.savez_compressed(HERE / "slices.npz", **store)


GEMM_CASES = [
    # name, m, n, k, phi, type2, type3, k_block, emu, max_slices, order, seed
    ("base_e4m3", 40, 36, 64, 0.5, "fp8e4m3", "fp32", 0, False, None, "smallest-first", 10),
    ("wide_e4m3", 24, 20, 48, 4.0, "fp8e4m3", "fp32", 0, False, None, "smallest-first", 11),
    ("emu_e4m3", 24, 24, 40, 0.5, "fp8e4m3", "fp32", 0, True, None, "smallest-first", 12),
    ("kblock_uneven", 20, 18, 100, 1.0, "fp8e4m3", "fp32", 64, False, None, "smallest-first", 13),
    ("kblock_emu", 16, 16, 90, 1.0, "fp16", "fp32", 32, True, None, "smallest-first", 14),
    ("fp16_base", 32, 30, 80, 2.0, "fp16", "fp32", 0, False, None, "smallest-first", 15),
    ("max_slices3", 20, 20, 64, 0.5, "fp8e4m3", "fp32", 0, False, 3, "smallest-first", 16),
    ("largest_first", 20, 22, 50, 0.5, "fp8e4m3", "fp32", 0, False, None, "largest-first", 17),
    ("type3_fp16", 16, 16, 32, 0.5, "fp8e4m3", "fp16", 0, False, None, "smallest-first", 18),
    ("bf16_base", 16, 18, 40, 0.5, "bf16", "fp32", 0, False, None, "smallest-first", 19),
    ("e5m2_base", 16, 18, 40, 0.5, "fp8e5m2", "fp32", 0, False, None, "smallest-first", 20),
    ("tall_thin", 130, 3, 17, 1.0, "fp8e4m3", "fp32", 0, False, None, "smallest-first", 21),
]


def gen_gemm():
    store = {}
    for name, m, n, k, phi, t2, t3, kbk, emu, ms, order, seed in GEMM_CASES:
        rng = np.random.default_rng(seed)
        A = spread(rng, m, k, phi)
        B = spread(rng, k, n, phi)
        A[2, :] = 0.0
        B[:, 1] = 0.0
        cfg = R.GemmConfig(R.get_format(t2), R.get_format(t3), k_block=kbk, fp64_emulation=emu,
                           max_slices=ms, accumulation_order=order)
        res = R.oz_gemm(A, B, cfg)
        store[f"{name}/A"] = A
        store[f"{name}/B"] = B
        store[f"{name}/C"] = res.C.view(np.uint64)
        store[f"{name}/blocks"] = np.array([[b.k_lo, b.k_hi, b.s_x, b.s_y, b.gemms] for b in res.stats.blocks],
                                           dtype=np.int64)
        store[f"{name}/cfg"] = np.array(json.dumps({"type2": t2, "type3": t3, "k_block": kbk, "emu": emu,
                                                    "max_slices": ms, "order": order}))
        st = res.stats
        store[f"{name}/ops"] = np.array([st.gemm_count, st.slicing_ops, st.gemm_ops, st.accum_ops], dtype=np.int64)
        print(name, [(b.s_x, b.s_y) for b in res.stats.blocks], flush=True)
    # exact small cases (tests/test_ozgemm.py:42-51 style)
    I = np.eye(8)
    X = spread(np.random.default_rng(30), 8, 8, 1.0)
    cfg = R.GemmConfig(R.get_format("fp8e4m3"), R.get_format("fp32"))
    store["identity/A"], store["identity/B"] = I, X
    store["identity/C"] = R.oz_gemm(I, X, cfg).C.view(np.uint64)
    store["scalar/A"], store["scalar/B"] = np.array([[1.5]]), np.array([[2.5]])
    store["scalar/C"] = R.oz_gemm(np.array([[1.5]]), np.array([[2.5]]), cfg).C.view(np.uint64)
    A = np.array([[1e16, 1.0, -1e16]])
    B = np.ones((3, 1))
    store["cancel/A"], store["cancel/B"] = A, B
    store["cancel/C"] = R.oz_gemm(A, B, cfg).C.view(np.uint64)
    np.savez_compressed(HERE / "gemm.npz", **store)


def gen_errors():
    out = {}
    f8, f32 = R.get_format("fp8e4m3"), R.get_format("fp32")
    cases = {
        "nan_input": (np.array([[1.0, np.nan]]), np.ones((2, 1)), R.GemmConfig(f8, f32)),
        "inf_input_B": (np.ones((1, 2)), np.array([[1.0], [np.inf]]), R.GemmConfig(f8, f32)),
        "subnormal_input": (np.array([[1.0, 5e-324]]), np.ones((2, 1)), R.GemmConfig(f8, f32)),
        "shape_mismatch": (np.ones((2, 3)), np.ones((2, 3)), R.GemmConfig(f8, f32)),
        "kblock_gt_k": (np.ones((2, 3)), np.ones((3, 2)), R.GemmConfig(f8, f32, k_block=4)),
    }
    for name, (A, B, cfg) in cases.items():
        try:
            R.oz_gemm(A, B, cfg)
            out[name] = None
        except Exception as e:  # noqa: BLE001
            out[name] = [type(e).__name__, [c.__name__ for c in type(e).__mro__]]
    for name, kw in {"kblock_neg": {"k_block": -1}, "max_slices0": {"max_slices": 0},
                     "bad_order": {"accumulation_order": "random"}}.items():
        try:
            R.GemmConfig(f8, f32, **kw)
            out[name] = None
        except Exception as e:  # noqa: BLE001
            out[name] = [type(e).__name__, [c.__name__ for c in type(e).__mro__]]
    (HERE / "errors.json").write_text(json.dumps(out, indent=1))


def gen_emu():
    vals = np.array([0.0, -0.0, 1.0, -1.0, 1.5, 2.0 ** -1022, -(2.0 ** -1022), 2.0 ** 1023, 3.0,
                     1.0 + 2.0 ** -52, 1.0 - 2.0 ** -53, 1e300, -1e300, 1e-300, 0.1, -0.3, 2.0 ** 52, 1.75])
    a, b = np.meshgrid(vals, vals)
    a, b = a.ravel(), b.ravel()
    res, ok = [], []
    for x, y in zip(a, b):
        try:
            r = fp64emu.add_arrays(np.array([x]), np.array([y]))[0]
            res.append(r)
            ok.append(True)
        except fp64emu.RangeError:
            res.append(0.0)
            ok.append(False)
    rng = np.random.default_rng(99)
    bitsr = (rng.integers(823, 1224, size=(2, 20000)).astype(np.uint64) << np.uint64(52)) \
        | rng.integers(0, 1 << 52, size=(2, 20000), dtype=np.int64).astype(np.uint64) \
        | (rng.integers(0, 2, size=(2, 20000)).astype(np.uint64) << np.uint64(63))
    ra, rb = bitsr[0].view(np.float64), bitsr[1].view(np.float64)
    np.savez_compressed(HERE / "emu_add.npz", a=a.view(np.uint64), b=b.view(np.uint64),
                        r=np.array(res).view(np.uint64), ok=np.array(ok),
                        ra=ra.view(np.uint64), rb=rb.view(np.uint64),
                        rr=fp64emu.add_arrays(ra, rb).view(np.uint64))


def gen_errors_ext():
    """errors_ext.json: what the reference raises (class name) or returns
    (sha256 of the C bits) for every case in error_cases.py."""
    import hashlib

    sys.path.insert(0, str(HERE))
    from error_cases import cases

    out = {}
    for name, (A, B, kw) in cases().items():
        kw = dict(kw)
        cfg = R.GemmConfig(R.get_format(kw.pop("type2")), R.get_format(kw.pop("type3")), **kw)
        try:
            C = R.oz_gemm(A, B, cfg).C
            out[name] = ["ok", hashlib.sha256(np.ascontiguousarray(C).view(np.uint64).tobytes()).hexdigest()]
        except Exception as e:  # noqa: BLE001
            out[name] = ["raise", type(e).__name__]
    (HERE / "errors_ext.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1:] == ["errors_ext"]:
        gen_errors_ext()
        raise SystemExit
    gen_params()
    gen_slices()
    gen_gemm()
    gen_errors()
    gen_emu()
    gen_errors_ext()
    print("golden fixtures written to", HERE)
