import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture
def lfopt():
    """Set library options (include/lfattn.h LF_OPT_*) for one test; restored after.
    The library reads its environment knobs once, so tests cannot use setenv."""
    from paper_2602_04789_b200 import _lib as L
    saved = []

    def set_(name, value):
        saved.append((name, L.set_option(name, int(value))))

    yield set_
    for name, prev in reversed(saved):
        L.set_option(name, prev)
