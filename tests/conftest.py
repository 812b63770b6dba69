"""Shared pytest setup.

Markers: ``gpu`` -- needs a B200 (run with ``-m gpu`` on the GPU box);
everything else runs on the CPU build container (``-m "not gpu"``).
"""

import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
for p in (REPO, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(HERE, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running test")


def pytest_collection_modifyitems(config, items):
    # a -m gpu run on a box without a device must fail loudly, not skip
    pass


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "small.npz"))


@pytest.fixture(scope="session")
def golden_cases():
    import json

    with open(os.path.join(GOLDEN, "cases.json")) as f:
        return json.load(f)
