import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the CUDA path through the C ABI")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """gcc pieces always; the nvcc pieces (libsd, synth CUDA) when stale or missing."""
    import __graft_entry__ as g

    g.build_host()
    try:
        g.build_cuda()
    except Exception as e:  # nvcc missing: host-only tests still run; GPU tests will fail loudly
        print(f"[conftest] CUDA build skipped: {e}")
    yield


def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
