"""The C-ABI library builds, loads and exports every symbol include/muxflow.h
declares.  CPU only: no compute calls (there is no GPU in the build box)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2303_13803_b200 import _native
from paper_2303_13803_b200 import build as nbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "muxflow.h")


def header_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(mux_\w+)\s*\(", src, re.M)))


def test_library_builds_and_loads():
    path = nbuild.build()
    assert os.path.exists(path)
    lib = _native.load()
    assert lib.mux_version().decode().startswith("muxflow")


def test_exports_every_declared_symbol():
    declared = header_functions()
    assert set(declared) == set(_native.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (mux_\w+)", out))
    missing = set(declared) - exported
    assert not missing, f"missing exports: {missing}"


def test_sm100a_code_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_table_validation_without_gpu():
    lib = _native.load()
    import numpy as np
    good = ((0.0, 0.5, 1.0), (0.5, 1.0), (0.0, 1.0))
    vals = np.linspace(0, 1, 12).reshape(3, 2, 2)
    vals = np.sort(vals, axis=2)
    tb, keep = _native.table_struct(good, vals)
    assert lib.mux_table_validate(ctypes.byref(tb)) == _native.MUX_OK
    bad = ((0.0, 0.0, 1.0), (0.5, 1.0), (0.0, 1.0))
    tb, keep = _native.table_struct(bad, vals)
    assert lib.mux_table_validate(ctypes.byref(tb)) == _native.MUX_EINVAL
    assert "strictly increasing" in lib.mux_last_error().decode()
    dip = vals.copy()
    dip[0, 0] = [0.5, 0.4]
    tb, keep = _native.table_struct(good, dip)
    assert lib.mux_table_validate(ctypes.byref(tb)) == _native.MUX_EINVAL


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2303_13803_b200 import default_table, predict_point
    with pytest.raises(RuntimeError):
        predict_point(default_table(), 0.5, 0.75, 0.5)
