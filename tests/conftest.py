import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfastmnmf.so")


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def rel(a, b):
    """Norm-wise relative error ||a - b||_F / ||b||_F (SURVEY §7 tolerance definition)."""
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (nb if nb > 0 else 1.0))


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)
