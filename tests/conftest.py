import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built liblfmm.so")
    config.addinivalue_line("markers", "slow: long-running (large systems)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def relerr(a, b):
    """max|a-b| / max|b| — the reference's own normalisation (bench.py:46-52)."""
    a = np.asarray(a)
    b = np.asarray(b)
    s = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / s if b.size else 0.0


@pytest.fixture(scope="session")
def golden():
    return load_golden
