"""Pin the CPU oracle to the reference: its outputs must equal, bit for bit,
the golden vectors produced by running ozdgemm 1.0.0 itself
(tests/golden/gen_golden.py)."""

import json
from pathlib import Path

import numpy as np
import pytest

import oracle

GOLD = Path(__file__).resolve().parent / "golden"


def _cases(npz):
    return sorted({k.split("/")[0] for k in npz.files})


SL = np.load(GOLD / "slices.npz")
GM = np.load(GOLD / "gemm.npz")


@pytest.mark.parametrize("name", _cases(SL))
def test_oracle_slices_match_reference(name):
    M = SL[f"{name}/M"]
    s_ref, rho, k = (int(v) for v in SL[f"{name}/meta"])
    orient = "cols" if "_cols" in name else "rows"
    emu = name.endswith("_emu")
    coeff, expo, s, flags = oracle.slice_matrix(M, orient, rho, emu)
    assert flags == 0
    assert s == s_ref
    assert np.array_equal(np.stack(coeff).view(np.uint64), SL[f"{name}/coeff"])
    assert np.array_equal(np.stack(expo), SL[f"{name}/expo"])


@pytest.mark.parametrize("name", [c for c in _cases(GM) if GM.__contains__(f"{c}/cfg")])
def test_oracle_gemm_matches_reference(name):
    cfg = json.loads(str(GM[f"{name}/cfg"]))
    C, info = oracle.oz_gemm(GM[f"{name}/A"], GM[f"{name}/B"], cfg["type2"], cfg["type3"], cfg["k_block"],
                             cfg["emu"], cfg["max_slices"], cfg["order"])
    assert info["flags"] == 0
    assert np.array_equal(C.view(np.uint64), GM[f"{name}/C"])
    assert [list(b) for b in info["blocks"]] == [list(r[:4]) for r in GM[f"{name}/blocks"]]


@pytest.mark.parametrize("name", ["identity", "scalar", "cancel"])
def test_oracle_exact_cases(name):
    C, info = oracle.oz_gemm(GM[f"{name}/A"], GM[f"{name}/B"])
    assert np.array_equal(C.view(np.uint64), GM[f"{name}/C"])


def test_oracle_emu_add_matches_reference():
    E = np.load(GOLD / "emu_add.npz")
    for a, b, r, ok in zip(E["a"], E["b"], E["r"], E["ok"]):
        got, flags = oracle.emu_add(float(a.view(np.float64)), float(b.view(np.float64)))
        if ok:
            assert flags == 0
            assert np.array([got]).view(np.uint64)[0] == r
        else:
            assert flags != 0
    # bulk random operands (fp64emu.add_arrays == hardware RNE there)
    for a, b, r in list(zip(E["ra"], E["rb"], E["rr"]))[:4000]:
        got, flags = oracle.emu_add(float(a.view(np.float64)), float(b.view(np.float64)))
        assert flags == 0 and np.array([got]).view(np.uint64)[0] == r


def test_oracle_emu_equals_hw():
    rng = np.random.default_rng(0)
    A = (rng.random((20, 90)) - 0.5) * np.exp(3 * rng.standard_normal((20, 90)))
    B = (rng.random((90, 17)) - 0.5) * np.exp(3 * rng.standard_normal((90, 17)))
    C1, _ = oracle.oz_gemm(A, B, emu=False)
    C2, _ = oracle.oz_gemm(A, B, emu=True)
    assert np.array_equal(C1.view(np.uint64), C2.view(np.uint64))


def test_oracle_config1_matches_reference():
    """BASELINE config 1 (n = 1024, phi = 0.5, reference defaults): the oracle's
    C has the sha256 of the C ozdgemm itself computed (gen_big_golden.py)."""
    import hashlib

    g = json.loads((GOLD / "config1.json").read_text())
    n, phi = g["n"], g["phi"]
    rng = np.random.default_rng(g["seed"])
    A = (rng.random((n, n)) - 0.5) * np.exp(phi * rng.standard_normal((n, n)))
    B = (rng.random((n, n)) - 0.5) * np.exp(phi * rng.standard_normal((n, n)))
    C, info = oracle.oz_gemm(A, B, g["type2"], g["type3"])
    assert info["flags"] == 0 and [list(b) for b in info["blocks"]] == g["blocks"]
    assert hashlib.sha256(C.view(np.uint64).tobytes()).hexdigest() == g["sha256_C"]


@pytest.mark.parametrize("key", ["64_1", "64_2", "64_3", "256_1", "512_2"])
def test_dd_checker_matches_reference_ref_gemm(key):
    """The double-double checker used for acceptance criteria 6/7 equals the
    reference's exact ref_gemm bit for bit on the criteria's inputs, and the
    naive restatement reproduces naive_gemm_fp64's error (golden accept.json)."""
    import hashlib

    meta = json.loads((GOLD / "accept.json").read_text())
    n, seed = (int(v) for v in key.split("_"))
    rng = np.random.default_rng(seed)
    A = 1.0 + 9.0 * rng.random((n, n))
    B = 1.0 + 9.0 * rng.random((n, n))
    C = oracle.dd_gemm(A, B)
    assert hashlib.sha256(C.view(np.uint64).tobytes()).hexdigest() == meta["hashes"][key]
    err = float(np.max(np.abs(oracle.naive_gemm(A, B) - C) / np.abs(C)))
    assert err == meta["err_naive"][key]
