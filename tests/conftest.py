import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def ak():
    import paper_2507_16710_b200 as ak_mod
    return ak_mod


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle


@pytest.fixture(scope="session")
def ex(ak):
    return ak.ExecBackend.cuda(0)


@pytest.fixture(scope="session")
def dev():
    import torch
    return torch.device("cuda:0")
