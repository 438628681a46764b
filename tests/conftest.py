"""Shared fixtures: golden vectors recorded from the reference, marker registration."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built native library")
    config.addinivalue_line("markers", "slow: large inputs (minutes on CPU)")


@pytest.fixture(scope="session")
def small_golden():
    arrays = np.load(os.path.join(GOLDEN, "small.npz"))
    with open(os.path.join(GOLDEN, "small.json")) as fh:
        meta = json.load(fh)
    return arrays, meta


@pytest.fixture(scope="session")
def large_golden():
    path = os.path.join(GOLDEN, "large.json")
    if not os.path.exists(path):
        pytest.skip("large goldens not recorded")
    with open(path) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def mrd_golden():
    arrays = np.load(os.path.join(GOLDEN, "mrd.npz"))
    with open(os.path.join(GOLDEN, "mrd.json")) as fh:
        meta = json.load(fh)
    return arrays, meta
