import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")


@pytest.fixture(scope="session")
def m1500():
    from oracle import oracle as O
    return O.load_coefficients("M1500")


@pytest.fixture(scope="session")
def m40():
    from oracle import oracle as O
    return O.load_coefficients("M40")
