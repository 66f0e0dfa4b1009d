import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture
def test_hook():
    """Set a library test hook (f46_set_test_hook) for one test; every hook
    set through it is reset to 0 afterwards."""
    from paper_2512_02010_b200 import _lib

    L = _lib.load()
    used = set()

    def set_hook(name, value):
        used.add(name)
        assert L.f46_set_test_hook(_lib.HOOK[name], int(value)) == 0

    yield set_hook
    for name in used:
        L.f46_set_test_hook(_lib.HOOK[name], 0)
