"""pytest configuration: the ``gpu`` marker and repo-root import path.

``-m "not gpu"`` runs here (no GPU): oracle pins, host logic, C-ABI symbol checks and
world-size-2 gloo tests.  ``-m gpu`` runs on a B200 and compares the CUDA path (through
the C-ABI) with the oracle.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# GPU test runs use a short device watchdog so a protocol bug fails fast instead of
# spinning for the default 30 s per call.
os.environ.setdefault("TORUS_TIMEOUT_MS", "5000")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have = torch.cuda.is_available()
        ngpu = torch.cuda.device_count() if have else 0
    except Exception:  # pragma: no cover
        have, ngpu = False, 0
    skip_gpu = pytest.mark.skip(reason="no CUDA device")
    skip_multi = pytest.mark.skip(reason="needs >= 2 CUDA devices")
    for item in items:
        if "gpu" in item.keywords and not have:
            item.add_marker(skip_gpu)
        if "multigpu" in item.keywords and ngpu < 2:
            item.add_marker(skip_multi)
