import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


def pytest_collection_modifyitems(config, items):
    # GPU tests are skipped loudly (not silently passed) when no GPU is present.
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device (run with gpurun)")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
