"""Shared test setup: markers, repo on sys.path, golden fixtures, GPU helpers."""

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def make_profile(sm, mem=0.3, iter_time=0.1):
    """Profile builder the reference's tests import from their conftest
    (/root/reference/pkg/tests/conftest.py:15-22); used by tests/ref_suite."""
    if os.path.join(ROOT, "pkg", "src") not in sys.path:
        sys.path.insert(0, os.path.join(ROOT, "pkg", "src"))
    from muxsim.core import WorkloadProfile
    return WorkloadProfile(sm_activity=sm, gpu_utilization=min(1.0, 1.8 * sm), sm_occupancy=0.5,
                           iter_time_separate=iter_time, mem_fraction=mem)


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
