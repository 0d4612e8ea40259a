import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a library")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        p = GOLDEN / name
        if not p.exists():
            pytest.skip(f"golden fixture {name} not generated")
        return np.load(p)
    return load


def worked_example():
    """Worked 4x4 of the reference tests (tests/helpers.py:23-28)."""
    x = np.zeros((4, 4), order="F")
    x[1, 0], x[2, 0], x[3, 0] = 2.0, 1.0, 3.0
    x[2, 1], x[3, 1] = 4.0, 1.0
    x[3, 2] = 5.0
    return x


def lower(a):
    return np.tril(np.asarray(a), -1)


EPS = np.finfo(np.float64).eps
