import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The reference compiled in place (only where /root/reference was mounted at build time)."""
    from oracle import REF_SO, Ref

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libref.so not built (reference not mounted at build time)")
    return Ref()


@pytest.fixture(scope="session")
def P():
    import paper_2208_06399_b200 as pkg

    return pkg


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
