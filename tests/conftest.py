import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) CUDA device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def kats():
    import json

    with open(os.path.join(GOLDEN, "reference_kats.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ref_vectors():
    import numpy as np

    return np.load(os.path.join(GOLDEN, "ref_vectors.npz"))


@pytest.fixture(scope="session")
def cuda():
    """The GPU tests must run the CUDA path; failing (not skipping) when the
    device is missing keeps a silent CPU pass impossible."""
    import torch

    from paper_1610_03618_b200 import capi

    assert torch.cuda.is_available(), "gpu test requires a CUDA device"
    assert capi.lib().lcnn_device_ok() == 1, "liblcnn_cuda.so needs an sm_100 device"
    return torch.device("cuda:0")
