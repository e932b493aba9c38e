import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built CUDA library")
    config.addinivalue_line("markers", "ref: needs oracle/_ref (the reference compiled from /root/reference)")


def pytest_collection_modifyitems(config, items):
    import oracle_lib
    if oracle_lib.ref_available():
        return
    skip = pytest.mark.skip(reason="oracle/_ref not built and /root/reference absent")
    for it in items:
        if "ref" in it.keywords:
            it.add_marker(skip)
