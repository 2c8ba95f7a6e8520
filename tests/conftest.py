"""Shared fixtures.  `-m gpu` tests need a B200 (sm_100a) and the in-tree
native library; everything else runs on CPU (oracle, host logic, ABI
surface, gloo multi-process)."""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def units():
    return load_golden("reference_units.npz")


@pytest.fixture(scope="session")
def small_runs():
    return load_golden("reference_small_runs.npz")


@pytest.fixture(scope="session")
def c0_ref():
    return load_golden("reference_c0.npz")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    O.set_mode("exact")
    return O


def reference_available():
    return os.path.isdir(REFERENCE_SRC)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
