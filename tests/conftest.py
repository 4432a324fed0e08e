import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for _p in (ROOT, TESTS):
    if _p not in sys.path:
        sys.path.insert(0, _p)
if False:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    """The C restatement (oracle/_build), pinned to the reference by
    tests/test_oracle_pin.py. Test infrastructure only."""
    from oracle import ffi
    return ffi.load("oracle")


@pytest.fixture(scope="session")
def ctx():
    from paper_1607_00531_b200.epicorr import Context
    return Context(0)
