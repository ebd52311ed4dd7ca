import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def load_golden(name):
    import numpy as np

    return dict(np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"), allow_pickle=False))


@pytest.fixture(scope="session")
def gpu_available():
    from paper_1305_6861_b200 import _capi

    _capi.load()
    return _capi.device_count() > 0
