import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running case")


def spread_matrix(rng, rows, cols, phi):
    """The north-star inputs: (rand - 0.5) * exp(phi * randn)."""
    return (rng.random((rows, cols)) - 0.5) * np.exp(phi * rng.standard_normal((rows, cols)))


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    return torch


@pytest.fixture
def pair_variant(cuda):
    """Force oz_pair_gemm's kernel variant for one test, then restore automatic."""
    from paper_2508_00441_b200 import _lib

    yield _lib.set_pair_variant
    _lib.set_pair_variant(0, 0, 0)
