import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libvmfa_b200.so")
    config.addinivalue_line("markers", "slow: full-size (BASELINE config) runs")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def vmfa():
    from paper_2501_12299_b200 import build as B
    B.build()
    from paper_2501_12299_b200 import vmfa as V
    return V


@pytest.fixture(scope="session")
def gpu(vmfa):
    if not vmfa.device_available():
        pytest.fail("gpu test without an sm_100 device: the CUDA path is required (no fallback)")
    return vmfa
