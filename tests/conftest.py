import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libfbgpu.so")
    config.addinivalue_line("markers", "slow: long-running (full-size configurations)")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN_DIR, "reference_golden.npz"))


@pytest.fixture(scope="session")
def golden_scalars():
    with open(os.path.join(GOLDEN_DIR, "reference_scalars.json")) as fh:
        return json.load(fh)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


@pytest.fixture
def random_image(rng):
    """Integer-valued 8-bit-range test image (same convention as the reference's conftest)."""
    def make(h, w, seed=None):
        r = rng if seed is None else np.random.default_rng(seed)
        return np.floor(r.uniform(0.0, 256.0, (h, w)))
    return make


@pytest.fixture(scope="session")
def tools_golden():
    """Reference outputs for I/O, metrology, convolve_direct and the CLI (make_golden_tools.py)."""
    return np.load(os.path.join(GOLDEN_DIR, "reference_tools.npz"))


@pytest.fixture(scope="session")
def tools_scalars():
    with open(os.path.join(GOLDEN_DIR, "reference_tools.json")) as fh:
        return json.load(fh)
