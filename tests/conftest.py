import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA path through the C-ABI library)")
    config.addinivalue_line("markers", "slow: full-size configs")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.fixture(scope="session")
def gold():
    return golden


@pytest.fixture(scope="session")
def lib():
    """The C-ABI library on a GPU box (skips nothing: GPU tests must fail
    loudly when the library or the device is missing)."""
    from paper_1907_06470_b200 import _lib

    return _lib.load()
