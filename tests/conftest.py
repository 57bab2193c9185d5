import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def pv1():
    from inputs import gen
    return gen.load_params("v1")


@pytest.fixture(scope="session")
def psym():
    from inputs import gen
    return gen.load_params("sym")


@pytest.fixture(scope="session")
def pgen():
    from inputs import gen
    return gen.load_params("generic")
