"""pytest configuration: the `gpu` marker and shared golden-fixture access.

`-m "not gpu"` runs here (no GPU): oracle-vs-golden, host logic, C-ABI
symbol checks, gloo multi-process tests.  `-m gpu` runs on a B200 and
exercises the CUDA path through the C ABI.
"""

import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the product kernels)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import get_oracle
    return get_oracle()


@pytest.fixture(scope="session")
def golden():
    from golden_io import Golden
    return Golden()
