import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs (run under torchrun)")


def _gpu_count() -> int:
    try:
        import torch

        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


def pytest_collection_modifyitems(config, items):
    n = _gpu_count()
    for it in items:
        if "gpu" in it.keywords and n == 0:
            it.add_marker(pytest.mark.skip(reason="no CUDA GPU"))


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle

    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import Oracle, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("reference")


def bits(a):
    """uint32 view for bitwise comparisons of float32 arrays."""
    return np.ascontiguousarray(a, np.float32).view(np.uint32)
