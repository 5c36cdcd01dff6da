"""Shared test setup: markers, repo on sys.path, golden fixtures, GPU helpers."""

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libmuxflow.so)")
    config.addinivalue_line("markers", "slow: larger sizes")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cuda():
    """The CUDA path must be live: fail (not skip) on a GPU test without it."""
    import torch
    assert torch.cuda.is_available(), "gpu-marked test needs a CUDA device"
    from paper_2303_13803_b200 import _native
    _native.load()
    torch.cuda.set_device(0)
    return torch
