import os
import sys

# Co-located multi-rank tests (tests/test_gpu_colocated.py) run N ranks'
# streams concurrently on one GPU: every stream needs its own hardware queue
# (embrace.h emb_shard_init_colocated).  Must be set before CUDA initialises.
os.environ["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"

import pytest  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: large-config test (minutes)")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
