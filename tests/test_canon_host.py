"""The canonicalisation's host loop (paper_2303_13803_b200/csrc/canon_host.h,
the reference's repair pass matching.py:173-199 over the tight graph) on tight
graphs recorded from real rounds on the B200 (MUX_TUNING=1 MUX_CANON_DUMP):
4k x 4k and 10k x 10k at 30 bits.  The recorded output is what the loop
emitted before the dead-row pruning; the pruned loop must emit the same
assignment.  CPU only: the harness is compiled with g++."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    exe = str(tmp_path_factory.mktemp("canon") / "canon_host_bench")
    subprocess.run([gxx, "-O2", "-std=c++17", "-I", os.path.join(ROOT, "paper_2303_13803_b200", "csrc"),
                    os.path.join(ROOT, "tools", "canon_host_bench.cpp"), "-o", exe], check=True)
    return exe


@pytest.mark.parametrize("name", ["canon_host_4k.bin", "canon_host_10k.bin"])
def test_host_loop_reproduces_recorded_assignment(harness, name):
    out = subprocess.run([harness, os.path.join(ROOT, "tests", "golden", name), "1"], capture_output=True, text=True)
    assert out.returncode == 0 and "output identical" in out.stdout, out.stdout + out.stderr
