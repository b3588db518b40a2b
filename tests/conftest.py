import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")


def _have_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def pcb_lib():
    """The in-tree C-ABI library; built on demand (nvcc is in the image on both sides)."""
    from paper_1805_06018_b200 import build, lib

    build.build()
    return lib.load()


@pytest.fixture(scope="session")
def gpu(pcb_lib):
    if not _have_gpu():
        pytest.fail("gpu-marked test run without a CUDA device")
    return pcb_lib
