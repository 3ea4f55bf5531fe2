import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libjv.so")


class Golden:
    """Reference-generated fixtures (tests/golden/make_golden.py)."""

    def __init__(self, path):
        self.z = np.load(path)
        self.names = [str(s) for s in self.z["_names"]]

    def case(self, name):
        pre = name + "/"
        return {k[len(pre):]: self.z[k] for k in self.z.files if k.startswith(pre)}


@pytest.fixture(scope="session")
def golden():
    return Golden(os.path.join(GOLDEN, "small.npz"))


def golden_names():
    z = np.load(os.path.join(GOLDEN, "small.npz"))
    return [str(s) for s in z["_names"]]


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)
