import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA path)")


@pytest.fixture(scope="session")
def hp():
    import paper_2205_03406_b200 as mod
    return mod


@pytest.fixture(scope="session")
def gpu_available():
    import paper_2205_03406_b200 as mod
    if mod.device_count() < 1:
        pytest.skip("no CUDA device")
    return True
