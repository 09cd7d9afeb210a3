import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large instances")


@pytest.fixture(scope="session")
def fg():
    import paper_2506_17471_b200 as m
    return m


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    return o
