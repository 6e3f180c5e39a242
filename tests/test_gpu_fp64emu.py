"""The device integer FP64 adds (emu_add = fp64emu.add_arrays' algorithm,
fast_add, and the emulated epilogue's add_lean) against IEEE binary64 RNE
(numpy) on random and adversarial operands: wide exponent ranges, every
exponent difference 0..70, near-total cancellation, power-of-two operands
with half-ulp-scale partners (the rounding-boundary cases), zeros."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(torch, a, b, mode):
    from paper_2508_00441_b200 import _lib

    ta = torch.from_numpy(a.view(np.int64).copy()).cuda()
    tb = torch.from_numpy(b.view(np.int64).copy()).cuda()
    out = torch.empty_like(ta)
    fl = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("oz_emu_add_batch", ta.data_ptr(), tb.data_ptr(), out.data_ptr(), a.size, mode, fl.data_ptr(),
              _lib.stream_ptr(torch))
    return out.cpu().numpy().view(np.uint64), int(fl.item())


def _cases(rng, n):
    sig = lambda k: rng.integers(0, 1 << 52, size=k, dtype=np.int64).astype(np.uint64)  # noqa: E731
    sgn = lambda k: rng.integers(0, 2, size=k).astype(np.uint64) << np.uint64(63)  # noqa: E731
    out = []
    # wide random normals
    e = rng.integers(300, 1700, size=(2, n)).astype(np.uint64)
    out.append(((e[0] << np.uint64(52)) | sig(n) | sgn(n), (e[1] << np.uint64(52)) | sig(n) | sgn(n)))
    # every exponent difference 0..70
    d = np.repeat(np.arange(71, dtype=np.uint64), n // 71 + 1)[:n]
    e0 = rng.integers(900, 1100, size=n).astype(np.uint64)
    out.append(((e0 << np.uint64(52)) | sig(n) | sgn(n), ((e0 - d) << np.uint64(52)) | sig(n) | sgn(n)))
    # near-total cancellation: b = -(a with a few low bits changed)
    a = (e0 << np.uint64(52)) | sig(n)
    b = (a ^ rng.integers(0, 1 << 8, size=n, dtype=np.int64).astype(np.uint64)) | np.uint64(1 << 63)
    out.append((a, b))
    # powers of two against partners around half / quarter ulp
    p2 = e0 << np.uint64(52)
    dd = rng.integers(50, 57, size=n).astype(np.uint64)
    out.append((p2 | sgn(n), ((e0 - dd) << np.uint64(52)) | sig(n) | sgn(n)))
    # FP32-significand terms (24 bits) against full-width accumulators, like Cb + G*2^e
    t = (e0 << np.uint64(52)) | ((sig(n) >> np.uint64(29)) << np.uint64(29)) | sgn(n)
    out.append(((rng.integers(850, 1150, size=n).astype(np.uint64) << np.uint64(52)) | sig(n) | sgn(n), t))
    # zeros
    z = np.zeros(n, dtype=np.uint64)
    out.append((z, a))
    out.append((a, z | np.uint64(1 << 63)))
    return out


@pytest.mark.parametrize("mode", [0, 1, 2], ids=["emu_add", "fast_add", "add_lean"])
def test_device_integer_adds_match_ieee(cuda, mode):
    torch = cuda
    rng = np.random.default_rng(123 + mode)
    for a, b in _cases(rng, 200_000):
        want = (a.view(np.float64) + b.view(np.float64)).view(np.uint64)
        got, fl = _run(torch, a, b, mode)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (mode, [(hex(int(a[i])), hex(int(b[i])), hex(int(got[i])), hex(int(want[i])))
                                      for i in bad[:4]])
        assert fl == 0


def test_device_mul_and_lt(cuda):
    """oz_emu_add_batch modes 3 / 4: integer-only multiply (fp64emu._mul_core,
    RNE incl. the carry into the next binade and exact ties) and the order
    compare (_lt_core: -0 == +0) against IEEE; range errors flagged."""
    torch = cuda
    rng = np.random.default_rng(11)
    n = 1 << 18
    sig = rng.integers(0, 1 << 52, size=(2, n), dtype=np.int64).astype(np.uint64)
    e = rng.integers(600, 1450, size=(2, n)).astype(np.uint64)
    s = rng.integers(0, 2, size=(2, n)).astype(np.uint64) << np.uint64(63)
    ab = (e << np.uint64(52)) | sig | s
    # significands that multiply to exact ties / all-ones carries
    ab[0, :1000] = (ab[0, :1000] & ~np.uint64((1 << 52) - 1)) | np.uint64((1 << 52) - 1)
    ab[1, :1000] = (ab[1, :1000] & ~np.uint64((1 << 52) - 1)) | np.uint64((1 << 52) - 1)
    ab[0, 1000:2000] = (ab[0, 1000:2000] & ~np.uint64((1 << 52) - 1)) | np.uint64(1 << 51)  # 1.5
    ab[1, 1000:2000] = (ab[1, 1000:2000] & ~np.uint64((1 << 52) - 1)) | np.uint64(1)        # 1 + ulp
    ab[0, 2000:2100] = np.uint64(0)
    ab[1, 2100:2200] = np.uint64(1 << 63)                                                     # -0
    a, b = ab[0].view(np.float64), ab[1].view(np.float64)
    got, fl = _run(torch, a, b, 3)
    assert fl == 0
    assert np.array_equal(got, (a * b).view(np.uint64))
    got, fl = _run(torch, a, b, 4)
    assert np.array_equal(got.astype(bool), a < b)
    # -0 < +0 is false both ways; equal operands are not less
    z = np.array([0.0, -0.0, 1.5], dtype=np.float64)
    got, _ = _run(torch, z, np.array([-0.0, 0.0, 1.5]), 4)
    assert not got.any()
    # out of the normal range: flagged (the reference raises RangeError)
    big = np.array([2.0 ** 600, 2.0 ** -600], dtype=np.float64)
    _, fl = _run(torch, big, big, 3)
    assert fl != 0
