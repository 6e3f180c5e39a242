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
