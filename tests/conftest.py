import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

# The library's default schedules commuting ops out of circuit order (within
# 1e-12 of the reference, not bit for bit). Most GPU tests pin the kernels
# bit for bit against the reference, so they run in circuit order; the
# default mode has its own tolerance tests (tests/test_gpu_reorder.py), which
# switch it on per environment (Env.set_ordering). Subprocess workers
# inherit this.
os.environ.setdefault("QGPU_ORDER", "exact")
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA product path)")
    config.addinivalue_line("markers", "slow: long-running (large states)")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the product library and the checkers once per session (nvcc and
    gcc cross-compile without a GPU)."""
    from paper_1802_08032_b200 import build as b

    b.build()
    import oracle

    oracle.build()
