import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) CUDA device")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


@pytest.fixture(scope="session")
def restated():
    from oracle.oracle import Restated

    return Restated()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import REF_SO, Reference

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libtgref.so not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def golden():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)
