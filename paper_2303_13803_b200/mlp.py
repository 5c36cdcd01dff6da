"""MLP speed-predictor plugin (the paper's predictor, absent from the reference).

The paper predicts co-location throughput with "four layers with hidden size
64x64" over online/offline workload features
and the SM share; the reference ships only a table and
says any regressor exported as a grid plugs in (predictor.py:6-8).  This
plugin evaluates the MLP itself for every pair on the GPU
(csrc/mlp.cu: layer 1 split into per-row / per-column partials, layers 2-3 as
tcgen05 fp16 GEMMs with split (hi + lo) activations and fp32 accumulation in
TMEM, ReLU and the final 64-wide dot fused into the TMEM->register
epilogues), either as a scoring call (`predict_pairs_mlp`), inside the GPU
round (`schedule(..., table=<MlpPredictor>)` -> `mux_round_mlp`), or exported
as a `PredictionTable` (`export_table`, the reference's plug-in hook
build_table_from_model, predictor.py:134-153).

Network (reading "four layers" as in -> 64 -> 64 -> 64 -> 1):
    x  = ([online(4), offline(4), share] - shift) * scale
    h1 = relu(W1 x + b1); h2 = relu(W2 h1 + b2); h3 = relu(W3 h2 + b3)
    w  = clamp(w4 . h3 + b4, 0, 1)
Features per workload: (gpu_utilization, sm_activity, sm_occupancy,
iter_time_separate).  The tensor-core layers' parameters (W2, b2, W3, b3) are
stored as fp16 values -- the model's deployment precision; the float64 oracle
(oracle/mlp_ref.py) uses the same stored values.  Training is out of scope
(SPEC.md:14); weights are supplied by the caller or drawn by
`MlpPredictor.random`.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat

HIDDEN = 64
N_FEAT = 9
FP16_PARAMS = ("W2", "b2", "W3", "b3")


def profile_features(p):
    """(gpu_utilization, sm_activity, sm_occupancy, iter_time_separate)."""
    return (p.gpu_utilization, p.sm_activity, p.sm_occupancy, p.iter_time_separate)


class MuxMlp(ctypes.Structure):
    _fields_ = [(name, ctypes.POINTER(ctypes.c_float)) for name in
                ("W1", "b1", "W2", "b2", "W3", "b3", "w4", "shift", "scale")] + \
               [("b4", ctypes.c_float), ("hidden", ctypes.c_int32)]


@dataclass(frozen=True)
class MlpPredictor:
    W1: np.ndarray      # [64, 9]
    b1: np.ndarray      # [64]
    W2: np.ndarray      # [64, 64]
    b2: np.ndarray
    W3: np.ndarray      # [64, 64]
    b3: np.ndarray
    w4: np.ndarray      # [64]
    b4: float
    shift: np.ndarray   # [9]
    scale: np.ndarray   # [9]
    gpu_type: str = "default"

    kind = "mlp"

    def __post_init__(self):
        shapes = {"W1": (HIDDEN, N_FEAT), "b1": (HIDDEN,), "W2": (HIDDEN, HIDDEN), "b2": (HIDDEN,),
                  "W3": (HIDDEN, HIDDEN), "b3": (HIDDEN,), "w4": (HIDDEN,), "shift": (N_FEAT,),
                  "scale": (N_FEAT,)}
        for name, shape in shapes.items():
            a = np.array(getattr(self, name), dtype=np.float32)
            if a.shape != shape:
                raise ValueError(f"MLP parameter {name} has shape {a.shape}, expected {shape}")
            if not np.all(np.isfinite(a)):
                raise ValueError(f"MLP parameter {name} has non-finite entries")
            if name in FP16_PARAMS:
                a = a.astype(np.float16).astype(np.float32)   # the tensor-core layers' stored precision
                if not np.all(np.isfinite(a)):
                    raise ValueError(f"MLP parameter {name} overflows fp16")
            a.setflags(write=False)
            object.__setattr__(self, name, a)
        object.__setattr__(self, "b4", float(np.float32(self.b4)))

    @classmethod
    def random(cls, seed=0):
        """He-initialised weights with a spread of outputs inside (0, 1)."""
        rng = np.random.default_rng(seed)
        he = lambda fan_in, shape: rng.normal(0.0, np.sqrt(2.0 / fan_in), shape)
        shift = np.array([0.5, 0.5, 0.5, 0.05, 0.8, 0.8, 0.5, 0.1, 0.4])
        scale = np.array([2.0, 2.0, 2.0, 20.0, 4.0, 4.0, 2.0, 10.0, 3.0])
        return cls(W1=he(N_FEAT, (HIDDEN, N_FEAT)), b1=rng.normal(0, 0.1, HIDDEN),
                   W2=he(HIDDEN, (HIDDEN, HIDDEN)), b2=rng.normal(0, 0.1, HIDDEN),
                   W3=he(HIDDEN, (HIDDEN, HIDDEN)), b3=rng.normal(0, 0.1, HIDDEN),
                   w4=rng.normal(0, 0.35 / np.sqrt(HIDDEN), HIDDEN), b4=0.5,
                   shift=shift, scale=scale)

    def params(self):
        return {k: getattr(self, k) for k in ("W1", "b1", "W2", "b2", "W3", "b3", "w4", "b4",
                                              "shift", "scale")}

    def struct(self):
        fp = ctypes.POINTER(ctypes.c_float)
        arrs = {k: np.ascontiguousarray(getattr(self, k), dtype=np.float32)
                for k in ("W1", "b1", "W2", "b2", "W3", "b3", "w4", "shift", "scale")}
        s = MuxMlp(*[arrs[k].ctypes.data_as(fp) for k in
                     ("W1", "b1", "W2", "b2", "W3", "b3", "w4", "shift", "scale")],
                   self.b4, HIDDEN)
        return s, arrs


def predict_pairs_mlp(mlp: MlpPredictor, on_feat, share, off_feat, dtype="float32", qbits=20, out=None):
    """GPU MLP scores for every (online u, offline v) pair.

    on_feat [N, 4] and off_feat [M, 4] (profile_features order), share [N].
    Returns a torch tensor [N, M] (float32 scores, or int32 rint(w * 2^qbits)
    with the 1e-6 edge floor) on the current CUDA device.
    """
    torch = nat.torch_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())

    def to_dev(a, shape1=None):
        t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a, dtype=np.float64))
        t = t.to(device=dev, dtype=torch.float64).contiguous()
        return t

    on = to_dev(on_feat).reshape(-1, 4)
    off = to_dev(off_feat).reshape(-1, 4)
    sh = to_dev(share).reshape(-1)
    n, m = on.shape[0], off.shape[0]
    if sh.shape[0] != n:
        raise ValueError("on_feat and share must have the same length")
    wtype, tdt = {"float32": (nat.MUX_W_F32, torch.float32), "int32": (nat.MUX_W_I32, torch.int32)}[dtype]
    ldo = max(4, ((m + 3) // 4) * 4)
    if out is None:
        out = torch.empty((n, ldo), dtype=tdt, device=dev)
    st, keep = mlp.struct()
    lib = nat.load()
    nat.check(lib.mux_score_mlp(nat.context(), ctypes.byref(st), on.data_ptr(), sh.data_ptr(), n,
                                off.data_ptr(), m, wtype, int(qbits), out.data_ptr(), ldo, nat.stream_ptr()))
    del keep
    return out[:, :m]


def export_table(mlp: MlpPredictor, online_sm=None, offline_sm=None, sm_pct=None, online_iter=0.02,
                 offline_iter=0.1, occupancy=0.5, gpu_type="default"):
    """The MLP sampled on a prediction grid: a `PredictionTable` the
    reference's table path accepts unchanged (its plug-in contract,
    predictor.py:6-8 and build_table_from_model, predictor.py:134-153).

    Grid point (x, y, z) = (online SM activity, offline SM activity, share);
    the other profile features follow the synthetic records (gpu_utilization
    = min(1, 1.8 sm), sm_occupancy = `occupancy`, iter_time_separate =
    `online_iter` / `offline_iter`).  All grid points are scored in one GPU
    call.  The table contract requires values non-decreasing along sm_pct
    (predictor.py:56-71), so the export takes the running maximum along that
    axis (a no-op for a monotone model)."""
    from .predictor import PredictionTable
    from .tables import DEFAULT_OFFLINE_SM, DEFAULT_ONLINE_SM, DEFAULT_SM_PCT
    xs = np.asarray(DEFAULT_ONLINE_SM if online_sm is None else online_sm, dtype=np.float64)
    ys = np.asarray(DEFAULT_OFFLINE_SM if offline_sm is None else offline_sm, dtype=np.float64)
    zs = np.asarray(DEFAULT_SM_PCT if sm_pct is None else sm_pct, dtype=np.float64)
    X, Z = np.meshgrid(xs, zs, indexing="ij")                  # rows = (x, z) pairs
    X, Z = X.reshape(-1), Z.reshape(-1)
    on = np.stack([np.minimum(1.0, 1.8 * X), X, np.full_like(X, occupancy), np.full_like(X, online_iter)], axis=1)
    off = np.stack([np.minimum(1.0, 1.8 * ys), ys, np.full_like(ys, occupancy), np.full_like(ys, offline_iter)], axis=1)
    W = predict_pairs_mlp(mlp, on, Z, off).cpu().numpy().astype(np.float64)   # [(x, z), y]
    vals = W.reshape(xs.size, zs.size, ys.size).transpose(0, 2, 1)            # [x][y][z]
    vals = np.maximum.accumulate(np.clip(vals, 0.0, 1.0), axis=2)
    return PredictionTable(online_sm=tuple(float(v) for v in xs), offline_sm=tuple(float(v) for v in ys),
                           sm_pct=tuple(float(v) for v in zs), values=vals, gpu_type=gpu_type)


def round_arrays_mlp(mlp: MlpPredictor, on_feat, share, off_feat, qbits=30, stats=False):
    """One GPU round with the MLP as the predictor (C ABI `mux_round_mlp`):
    host features in, MLP scores quantised to 30-bit weights in HBM, the
    exact matching, col_of_row out (-1 = unmatched).  Returns (col, total_q[,
    stats])."""
    nat.torch_cuda()
    on = np.ascontiguousarray(np.asarray(on_feat, dtype=np.float64).reshape(-1, 4))
    off = np.ascontiguousarray(np.asarray(off_feat, dtype=np.float64).reshape(-1, 4))
    sh = np.ascontiguousarray(np.asarray(share, dtype=np.float64).reshape(-1))
    n, m = on.shape[0], off.shape[0]
    if sh.shape[0] != n:
        raise ValueError("on_feat and share must have the same length")
    col = np.empty(max(n, 1), dtype=np.int32)
    total = ctypes.c_int64(0)
    st = nat.MuxStats()
    s, keep = mlp.struct()
    dp = ctypes.c_void_p
    nat.check(nat.load().mux_round_mlp(nat.context(), ctypes.byref(s), dp(on.ctypes.data), dp(sh.ctypes.data), n,
                                       dp(off.ctypes.data), m, int(qbits), dp(col.ctypes.data), ctypes.byref(total),
                                       ctypes.byref(st), nat.stream_ptr()))
    del keep
    if stats:
        return col[:n], int(total.value), st.as_dict()
    return col[:n], int(total.value)
