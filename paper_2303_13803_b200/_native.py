"""ctypes binding of libmuxflow.so (include/muxflow.h).

The CUDA library is the only compute path: if it is missing, or no B200 is
visible, every compute entry point raises -- there is no CPU fallback.
Device buffers are torch tensors (plumbing only); the library sees raw
pointers and the current torch stream.
"""

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmuxflow.so")
if os.environ.get("MUX_TUNING") == "1" and os.environ.get("MUX_LIB_VARIANT"):
    # experiment builds (tools/build_variant.py): same sources, other compile-time constants
    LIB_PATH = os.path.join(_HERE, "..", "tools", "_variants", os.environ["MUX_LIB_VARIANT"] + ".so")

MUX_OK, MUX_EINVAL, MUX_ECUDA, MUX_ENOMEM, MUX_ELIMIT = 0, 1, 2, 3, 4
MUX_W_F64, MUX_W_F32, MUX_W_I32, MUX_W_I64 = 0, 1, 2, 3
MUX_SCORE_EXACT, MUX_SCORE_FAST = 0, 1

# every symbol include/muxflow.h declares (checked by tests/test_native_abi.py)
EXPORTS = ("mux_version", "mux_last_error", "mux_ctx_create", "mux_ctx_destroy",
           "mux_table_validate", "mux_score_table", "mux_score_mlp", "mux_match", "mux_match_keyed",
           "mux_round", "mux_round_dev", "mux_round_mlp", "mux_ipc_export", "mux_ipc_import")


class MuxTable(ctypes.Structure):
    _fields_ = [("n_online_sm", ctypes.c_int32), ("n_offline_sm", ctypes.c_int32),
                ("n_sm_pct", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("online_sm", ctypes.POINTER(ctypes.c_double)),
                ("offline_sm", ctypes.POINTER(ctypes.c_double)),
                ("sm_pct", ctypes.POINTER(ctypes.c_double)),
                ("values", ctypes.POINTER(ctypes.c_double))]


class MuxStats(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in
                ("n_rows", "n_cols", "n_square", "phases", "rounds", "bids", "row_scans",
                 "tail_bids", "total_q")] + \
               [("ms_score", ctypes.c_double), ("ms_match", ctypes.c_double),
                ("launches", ctypes.c_int64), ("ms_tail", ctypes.c_double),
                ("ms_kernel", ctypes.c_double), ("cache_hits", ctypes.c_int64),
                ("ms_canon", ctypes.c_double), ("canon_searches", ctypes.c_int64),
                ("tight_edges", ctypes.c_int64), ("dual_sweeps", ctypes.c_int64),
                ("levels", ctypes.c_int64), ("par_steps", ctypes.c_int64), ("dense_steps", ctypes.c_int64),
                ("dense_searches", ctypes.c_int64), ("ms_dense", ctypes.c_double),
                ("ms_parallel", ctypes.c_double), ("dense_bytes", ctypes.c_double),
                ("dense_launches", ctypes.c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class NativeError(RuntimeError):
    def __init__(self, status, message):
        super().__init__(f"muxflow status {status}: {message}")
        self.status = status
        self.message = message


_lib = None
_lock = threading.Lock()
_ctx = {}


def load():
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"muxflow CUDA library not built: {LIB_PATH} is missing "
                               "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
        lib = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        lib.mux_version.restype = ctypes.c_char_p
        lib.mux_last_error.restype = ctypes.c_char_p
        lib.mux_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(P)]
        lib.mux_ctx_destroy.argtypes = [P]
        lib.mux_table_validate.argtypes = [ctypes.POINTER(MuxTable)]
        lib.mux_score_table.argtypes = [P, ctypes.POINTER(MuxTable), P, P, i64, P, i64, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, P, i64, P]
        lib.mux_score_mlp.argtypes = [P, P, P, P, i64, P, i64, ctypes.c_int, ctypes.c_int, P, i64, P]
        lib.mux_match.argtypes = [P, P, ctypes.c_int, i64, i64, i64, P, ctypes.c_int,
                                  ctypes.POINTER(i64), ctypes.POINTER(MuxStats), P]
        lib.mux_match_keyed.argtypes = [P, P, ctypes.c_int, i64, i64, i64, P, P, P, ctypes.c_int,
                                        ctypes.POINTER(i64), ctypes.POINTER(MuxStats), P]
        lib.mux_round.argtypes = [P, ctypes.POINTER(MuxTable), P, P, i64, P, i64, ctypes.c_int, P,
                                  ctypes.POINTER(i64), ctypes.POINTER(MuxStats), P]
        lib.mux_round_dev.argtypes = [P, ctypes.POINTER(MuxTable), P, P, i64, P, i64, ctypes.c_int, P, i64, P,
                                      P, P, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(MuxStats), P]
        lib.mux_round_mlp.argtypes = [P, P, P, P, i64, P, i64, ctypes.c_int, P, ctypes.POINTER(i64),
                                      ctypes.POINTER(MuxStats), P]
        lib.mux_ipc_export.argtypes = [P, i64, ctypes.POINTER(P), P]
        lib.mux_ipc_import.argtypes = [P, P, ctypes.POINTER(P)]
        for name in EXPORTS[2:]:
            getattr(lib, name).restype = ctypes.c_int
        _lib = lib
    return _lib


def check(status):
    if status != MUX_OK:
        msg = load().mux_last_error().decode(errors="replace")
        raise NativeError(status, msg)


def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("muxflow needs a CUDA device (B200); none is visible")
    return torch


def context(device=None):
    """Per-device native context (created once, lives for the process)."""
    torch = torch_cuda()
    dev = torch.cuda.current_device() if device is None else int(device)
    c = _ctx.get(dev)
    if c is None:
        lib = load()
        h = ctypes.c_void_p()
        check(lib.mux_ctx_create(dev, ctypes.byref(h)))
        c = _ctx[dev] = h
    return c


def stream_ptr(device=None):
    torch = torch_cuda()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def table_struct(axes, values):
    """MuxTable over float64 numpy arrays; returns (struct, keepalive)."""
    import numpy as np
    ax = [np.ascontiguousarray(a, dtype=np.float64) for a in axes]
    vals = np.ascontiguousarray(values, dtype=np.float64)
    dp = ctypes.POINTER(ctypes.c_double)
    t = MuxTable(len(ax[0]), len(ax[1]), len(ax[2]), 0,
                 ax[0].ctypes.data_as(dp), ax[1].ctypes.data_as(dp), ax[2].ctypes.data_as(dp),
                 vals.ctypes.data_as(dp))
    return t, (ax, vals)
