import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large-size parity (minutes)")


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import Oracle
    return Oracle.get()


@pytest.fixture(scope="session")
def sp():
    import paper_2409_10743_b200 as sp
    return sp
