import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run under gpurun")


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    marker = config.getoption("-m") or ""
    if "gpu" in marker and "not gpu" not in marker:
        return  # explicit -m gpu without a device: let the tests fail loudly
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
