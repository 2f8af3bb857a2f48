import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through libhetm_b200.so on cuda:0)")
    config.addinivalue_line("markers", "slow: full BASELINE-size property checks")


@pytest.fixture(scope="session")
def hetm():
    import paper_1905_00661_b200 as h
    return h


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle
