import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a path")
    config.addinivalue_line("markers", "slow: long-running (large workloads)")
    config.addinivalue_line("markers", "large: BASELINE configs 3-5 at full size (run first)")


def pytest_collection_modifyitems(config, items):
    # the large-config parity tests run first, so that -x cannot hide them behind another failure
    items.sort(key=lambda it: 0 if "large" in it.keywords else 1)
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
