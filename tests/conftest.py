"""Shared test setup: the `gpu` marker, repo imports, golden fixtures."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU and the built libkvlinc.so")


@pytest.fixture(scope="session")
def golden():
    """Golden vectors produced by running the reference (tests/golden/make_golden.py)."""
    out = {}
    for name in ("quantize", "hadamard", "adapter", "cache", "attention", "train"):
        with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
            out[name] = {k: z[k] for k in z.files}
    return out
