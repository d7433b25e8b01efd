import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhekan_gpu.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu_lib():
    """Build (if needed) and load the product library; GPU tests only."""
    if not gpu_available():
        pytest.skip("no CUDA device")
    from paper_2409_07751_b200.build import build
    build()
    from paper_2409_07751_b200.engine import load_library
    return load_library()
