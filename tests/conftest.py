import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for _p in (TESTS, ROOT):
    if _p not in sys.path:
        sys.path.insert(0, _p)

from asse_testutil import read_golden  # noqa: E402,F401


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (parity tests through the C-ABI)")
    config.addinivalue_line("markers", "slow: long-running (still part of the suite)")


@pytest.fixture(scope="session")
def cuda_device():
    """GPU tests fail loudly (never skip) when CUDA is not usable."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu-marked test run without a usable CUDA device")
    return torch.device("cuda:0")
