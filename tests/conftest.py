import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running (large sizes)")


def pytest_collection_modifyitems(config, items):
    pass


@pytest.fixture(scope="session")
def fgt():
    import paper_1909_09825_b200 as m
    return m
