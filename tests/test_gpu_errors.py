"""Failure semantics of the CUDA path against the REFERENCE's own behaviour.

Every case of tests/golden/error_cases.py goes through ``oz_gemm`` on the GPU
(split flags, epilogue term-range flags, emulated range errors) and must raise
the exception class the reference raised on the same inputs, or return the
same C bits (tests/golden/errors_ext.json, produced by gen_golden.py running
ozdgemm itself).  Covers slicing.py:119-125, :155-158, ozgemm.py:132-140,
:147-154 and fp64emu.py:269-277, including the order in which the reference
raises (A before B; block by block).
"""

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLD))
from error_cases import cases  # noqa: E402

pytestmark = pytest.mark.gpu
EXPECTED = json.loads((GOLD / "errors_ext.json").read_text())
CASES = cases()


def _exc(oz, name):
    return {"ValueError": ValueError, "RangeError": oz.RangeError, "DimensionError": oz.DimensionError,
            "SlicingInfeasible": oz.SlicingInfeasible}[name]


@pytest.mark.parametrize("name", sorted(CASES))
def test_failure_semantics_match_reference(cuda, name):
    import paper_2508_00441_b200 as oz

    A, B, kw = CASES[name]
    kw = dict(kw)
    cfg = oz.GemmConfig(oz.get_format(kw.pop("type2")), oz.get_format(kw.pop("type3")), **kw)
    kind, what = EXPECTED[name]
    if kind == "raise":
        exc = _exc(oz, what)
        with pytest.raises(exc) as ei:
            oz.oz_gemm(A, B, cfg)
        # the exact class, not a subclass/superclass stand-in (DimensionError is a ValueError)
        assert type(ei.value).__name__ == what, f"{name}: raised {type(ei.value).__name__}, reference {what}"
    else:
        C = oz.oz_gemm(A, B, cfg).C
        assert hashlib.sha256(np.ascontiguousarray(C).view(np.uint64).tobytes()).hexdigest() == what


@pytest.mark.parametrize("name", [n for n in sorted(CASES) if n.startswith("term_") or n == "sigma_range"])
def test_failure_cases_device_tensors(cuda, name):
    """Same cases with CUDA tensors in (no host copies; deferred flag check)."""
    torch = cuda
    import paper_2508_00441_b200 as oz

    A, B, kw = CASES[name]
    kw = dict(kw)
    cfg = oz.GemmConfig(oz.get_format(kw.pop("type2")), oz.get_format(kw.pop("type3")), **kw)
    kind, what = EXPECTED[name]
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    if kind == "raise":
        with pytest.raises(_exc(oz, what)):
            oz.oz_gemm(Ad, Bd, cfg)
    else:
        C = oz.oz_gemm(Ad, Bd, cfg).C.cpu().numpy()
        assert hashlib.sha256(np.ascontiguousarray(C).view(np.uint64).tobytes()).hexdigest() == what


@pytest.mark.parametrize("fmt", ["fp8e4m3", "fp16", "bf16"])
@pytest.mark.parametrize("emu", [False, True])
@pytest.mark.parametrize("scale", [-500, -300, 300, 500])
def test_far_exponents_match_oracle(cuda, fmt, emu, scale):
    """Operands near 2^+-500 (terms near the ends of the FP64 range) in every
    slice format and both accumulation modes: C and the raised class agree with
    the CPU oracle (reference algorithm)."""
    import oracle
    import paper_2508_00441_b200 as oz

    rng = np.random.default_rng(abs(scale) + len(fmt) + emu)
    A = (rng.random((70, 96)) - 0.5) * np.exp(2.0 * rng.standard_normal((70, 96))) * 2.0 ** scale
    B = (rng.random((96, 50)) - 0.5) * np.exp(2.0 * rng.standard_normal((96, 50))) * 2.0 ** scale
    cfg = oz.GemmConfig(oz.get_format(fmt), oz.get_format("fp32"), fp64_emulation=emu)
    Cref, info = oracle.oz_gemm(A, B, fmt, "fp32", 0, emu)
    if info["flags"]:
        with pytest.raises(oz.RangeError):
            oz.oz_gemm(A, B, cfg)
    else:
        C = oz.oz_gemm(A, B, cfg).C
        assert np.array_equal(C.view(np.uint64), Cref.view(np.uint64))
