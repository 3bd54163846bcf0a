import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


@pytest.fixture(scope="session")
def golden_ops():
    import numpy as np
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "golden_ops.npz"), allow_pickle=False))


@pytest.fixture(scope="session")
def golden_recon():
    import numpy as np
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "golden_recon.npz"), allow_pickle=False))
