"""Shared pytest setup.

``gpu`` marks tests that need a real B200 (they call the CUDA library through
its C ABI); everything else runs on CPU here.
"""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    if not cuda_available():
        pytest.fail("gpu-marked test run without a CUDA device")
    import torch

    return torch.device("cuda:0")
