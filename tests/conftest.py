import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built libkcache_b200.so")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Restatement
    return Restatement()


@pytest.fixture(scope="session")
def kc():
    """The product API. On a GPU box a missing library or GPU is an error, not a skip."""
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2404_18057_b200 import kcache
    kcache.load()
    return kcache
