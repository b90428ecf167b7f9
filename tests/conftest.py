import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running check")


@pytest.fixture(scope="session")
def oracle():
    from oracle import pyoracle
    pyoracle.oracle_lib()
    return pyoracle


@pytest.fixture(scope="session")
def gpu():
    """The product API; the tests that use it are GPU-only and must run the
    CUDA library (no fallback exists)."""
    from paper_1904_00429_b200 import mlsketch, _lib
    if _lib.lib().mlsk_device_count() < 1:
        pytest.fail("no CUDA device visible to the library")
    return mlsketch
