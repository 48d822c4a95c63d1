import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run through gpurun)")


@pytest.fixture(scope="session")
def stage1():
    with np.load(os.path.join(GOLDEN, "stage1.npz")) as z:
        return {k: z[k] for k in z.files}


def bits_equal(a, b):
    """Bit-for-bit equality of float arrays (NaN == NaN)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))
