import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.build()
    return O


@pytest.fixture(scope="session")
def same_blas(oracle):
    """True when this host's BLAS dispatches to the kernel the fixtures were made with."""
    oracle.use_reference_blas(True)
    g = golden("solves")
    return str(g["corename"]) == oracle.blas_corename()


def assert_bits(a, b, msg=""):
    """Bitwise equality of float arrays (signed zeros and NaN payloads included)."""
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    assert a.shape == b.shape, (a.shape, b.shape, msg)
    assert np.array_equal(a.view(np.int64), b.view(np.int64)), msg
