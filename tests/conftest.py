import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")

# Constants of the reference test suite (reference tests/conftest.py:8-10).
TEST_PARAMS = dict(radius=6.37122e6, omega=7.292e-5, gravity=9.80616, nu=1.0e5, h_bar=29400.0)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running")


def rel_err(got, want):
    import numpy as np

    got = np.asarray(got)
    want = np.asarray(want)
    scale = np.max(np.abs(want))
    if scale == 0:
        return float(np.max(np.abs(got)))
    return float(np.max(np.abs(got - want)) / scale)
