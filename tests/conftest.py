import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def laiv():
    from paper_2502_20969_b200 import laiv as m

    return m


@pytest.fixture(autouse=True)
def _free_devices():
    """Device contexts own multi-GB HBM caches: collect them between tests."""
    yield
    import gc

    gc.collect()
