import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


GOLDEN = os.path.join(HERE, "golden")
GOLDEN_CASES = ["four_points", "two_clusters", "rand600_d16", "d384_m32", "d384_m64", "d64_m16",
                "ties_empty"]


def load_golden(name):
    import numpy as np
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    grid = [tuple(int(v) for v in g) for g in z["grid"]]
    return os.path.join(GOLDEN, name + ".pragix"), z, grid


@pytest.fixture(scope="session")
def golden():
    return load_golden
