import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (exhaustive / full-size) case")


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def golden():
    import json

    d = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    with open(os.path.join(d, "utf8_to_utf16.json")) as f:
        u8 = json.load(f)
    with open(os.path.join(d, "utf16_to_utf8.json")) as f:
        u16 = json.load(f)
    with open(os.path.join(d, "misc.json")) as f:
        misc = json.load(f)
    return {"u8": u8, "u16": u16, "misc": misc}


@pytest.fixture(scope="session")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch
