import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a library)")


def golden(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def cuda():
    """The device the gpu tests run on; fails loudly if the B200 path is absent."""
    import torch
    assert torch.cuda.is_available(), "gpu test without a CUDA device"
    from paper_1602_05650_b200 import _native
    _native.load(require_device=True)
    return torch.device("cuda:0")
