import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: large parity case")


@pytest.fixture(scope="session", autouse=True)
def _oracle_built():
    """The CPU checkers (oracle/) must exist; build them when the sources
    are present (this container). On the GPU box they arrive prebuilt."""
    import oracle
    if os.path.isdir(oracle.REFERENCE_SRC) or not os.path.exists(oracle.ORACLE_LIB):
        oracle.build()
    yield


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    torch.cuda.init()
    return torch.device("cuda:0")
