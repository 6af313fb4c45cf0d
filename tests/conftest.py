"""Shared test setup: the repo root on sys.path, the ``gpu`` marker, fixtures.

``-m "not gpu"`` tests run on CPU (oracle vs golden fixtures, host logic, ABI
load); ``-m gpu`` tests are the parity tests proper and call the CUDA engine
through the C ABI.  Fixtures under tests/golden/ were produced by the
unmodified reference (tests/golden/make_golden.py)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name))
    return load


@pytest.fixture(scope="session")
def engine():
    """Built + loaded engine with a live device context (GPU tests only)."""
    import __graft_entry__

    __graft_entry__.build()
    from paper_2604_13144_b200 import _lib

    _lib.context(0)
    return _lib
