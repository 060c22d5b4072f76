import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden2d():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "reference_2d.npz"))


@pytest.fixture(scope="session")
def golden_c1():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "c1_full.npz"))
