"""Run the reference's own hot-path tests (matching, predictor, scheduler;
/root/reference/pkg/tests, vendored verbatim as ref_*.py) against this
repo's drop-in `muxsim` package (pkg/src/muxsim), i.e. through
libmuxflow.so on the GPU.  Every test here is marked `gpu`.

The reference's shared conftest imports the simulator's suite runner (out of
scope); the one helper these three files use, `make_profile`, is defined
here (and in tests/conftest.py) with the reference's body
(/root/reference/pkg/tests/conftest.py:15-22).
"""

import os
import sys

import pytest

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
_PKG = os.path.join(_ROOT, "pkg", "src")
if _PKG not in sys.path:
    sys.path.insert(0, _PKG)


def make_profile(sm, mem=0.3, iter_time=0.1):
    from muxsim.core import WorkloadProfile
    return WorkloadProfile(sm_activity=sm, gpu_utilization=min(1.0, 1.8 * sm), sm_occupancy=0.5,
                           iter_time_separate=iter_time, mem_fraction=mem)


def pytest_collection_modifyitems(config, items):
    here = os.path.dirname(os.path.abspath(__file__))
    for it in items:
        if str(it.fspath).startswith(here):
            it.add_marker(pytest.mark.gpu)


@pytest.fixture(autouse=True)
def _drop_in_is_ours(request):
    """The `muxsim` under test must be this repo's shim, never the reference."""
    import muxsim
    assert os.path.abspath(muxsim.__file__).startswith(_PKG), muxsim.__file__
