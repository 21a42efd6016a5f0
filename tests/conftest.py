import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


# PyTorch first: its libnccl.so.2 may be newer than the system's, and the
# engine opens whichever libnccl.so.2 the process already has (sharded.cu).
try:
    import torch  # noqa: F401
except Exception:  # CPU box without a working torch import: nothing to order
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.Port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    return oracle.Ref()


@pytest.fixture(scope="session")
def lib():
    from paper_2309_14311_b200 import capi
    return capi.load()
