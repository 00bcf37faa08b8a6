"""Shared test setup.

Markers: ``gpu`` -- needs a CUDA device and the in-tree CUDA library (run on
the B200 box with ``pytest -m gpu``); everything else runs on CPU.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (ROOT, os.path.join(ROOT, "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the CUDA library")
    config.addinivalue_line("markers", "slow: BASELINE-size host work (tens of seconds)")


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """The C ABI library must exist (build() compiles it); build if stale."""
    from paper_2202_04140_b200 import build
    build.build()


@pytest.fixture(scope="session")
def golden():
    def load(name):
        path = os.path.join(GOLDEN, name)
        if name.endswith(".json"):
            with open(path) as fh:
                return json.load(fh)
        return dict(np.load(path, allow_pickle=False))
    return load


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test collected without a CUDA device")
    return torch.device("cuda", 0)
