import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: longer-running parity case")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    """Skip-free guard: -m gpu tests must run on a GPU box and fail loudly otherwise."""
    if not _has_gpu() and os.environ.get("NBX_ALLOW_NO_GPU") != "1":
        pytest.fail("GPU test collected on a machine without a CUDA device")
    from paper_2205_07976_b200 import _native

    return _native.context()
