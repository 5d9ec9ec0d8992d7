import os
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference, REF_PATH
    if not REF_PATH.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def fm():
    """The product API; GPU tests require it to be backed by a real device."""
    import paper_2205_10879_b200 as fm_mod
    from paper_2205_10879_b200 import _native
    if _native.LIB.fmgp_device_count() < 1:
        pytest.fail("GPU test ran without a CUDA device")
    return fm_mod
