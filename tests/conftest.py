import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: full-size configuration runs")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"golden_{name}.npz")))


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
