"""Shared pytest setup: the ``gpu`` marker and fixture helpers."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


_cache = {}


def golden(name):
    """Load tests/golden/<name>.npz once per session (produced by make_golden.py)."""
    if name not in _cache:
        with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as d:
            _cache[name] = {k: d[k] for k in d.files}
    return _cache[name]


@pytest.fixture(scope="session")
def gold():
    return golden
