"""Shared test plumbing.

Markers: `gpu` tests need a B200 (run with `-m gpu` on the GPU box); all others
run on CPU.  Golden fixtures under tests/golden/ were produced by running the
reference itself (tools/make_golden.py); the CPU oracle (oracle/) is test
infrastructure only.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLD = os.path.join(ROOT, "tests", "golden")

# Tolerance stated by north_star for floating-point features (BASELINE.json).
REL_TOL = 1e-6


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLD, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_arrays():
    return dict(np.load(os.path.join(GOLD, "masks_small.npz")))


@pytest.fixture(scope="session")
def golden_clouds():
    return dict(np.load(os.path.join(GOLD, "clouds.npz")))


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle

    oracle.lib()
    return oracle


def rel_err(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.fixture(scope="session")
def sc():
    import paper_2510_02894_b200 as pkg

    return pkg


@pytest.fixture
def cuda_device():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return 0
