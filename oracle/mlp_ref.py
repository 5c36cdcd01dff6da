"""Oracle for the MLP speed-predictor plugin (TEST INFRASTRUCTURE ONLY).

PARITY UNPINNED: the reference has no MLP.  The paper describes the predictor
as "four layers with hidden size 64x64" over
the online/offline workload features and the SM share; the
reference ships only the table predictor (predictor.py:6-8).  This module is a
float64 numpy forward pass of the exact network the CUDA plugin
(paper_2303_13803_b200/csrc/mlp.cu) evaluates, with the same weights:

    x   = [online(4), offline(4), share]  scaled by (x - shift) * scale
    h1  = relu(W1 x + b1)          64
    h2  = relu(W2 h1 + b2)         64
    h3  = relu(W3 h2 + b3)         64
    w   = clamp(w4 . h3 + b4, 0, 1)

Feature order per workload: (gpu_utilization, sm_activity, sm_occupancy,
iter_time_separate) -- the WorkloadProfile fields (core.py:30-46).
"""

import numpy as np


def forward(params, on_feat, share, off_feat):
    """Dense N x M forward in float64.  on_feat [N,4], share [N], off_feat [M,4]."""
    W1 = np.asarray(params["W1"], dtype=np.float64)       # [64, 9]
    b1 = np.asarray(params["b1"], dtype=np.float64)
    W2 = np.asarray(params["W2"], dtype=np.float64)       # [64, 64]
    b2 = np.asarray(params["b2"], dtype=np.float64)
    W3 = np.asarray(params["W3"], dtype=np.float64)
    b3 = np.asarray(params["b3"], dtype=np.float64)
    w4 = np.asarray(params["w4"], dtype=np.float64)       # [64]
    b4 = float(params["b4"])
    shift = np.asarray(params["shift"], dtype=np.float64)  # [9]
    scale = np.asarray(params["scale"], dtype=np.float64)  # [9]
    on = (np.asarray(on_feat, dtype=np.float64) - shift[:4]) * scale[:4]
    off = (np.asarray(off_feat, dtype=np.float64) - shift[4:8]) * scale[4:8]
    s = (np.asarray(share, dtype=np.float64) - shift[8]) * scale[8]
    P = on @ W1[:, :4].T + s[:, None] * W1[:, 8][None, :] + b1      # [N, 64]
    Q = off @ W1[:, 4:8].T                                          # [M, 64]
    N, M = P.shape[0], Q.shape[0]
    out = np.empty((N, M))
    for u in range(N):
        h1 = np.maximum(P[u][None, :] + Q, 0.0)          # [M, 64]
        h2 = np.maximum(h1 @ W2.T + b2, 0.0)
        h3 = np.maximum(h2 @ W3.T + b3, 0.0)
        out[u] = np.clip(h3 @ w4 + b4, 0.0, 1.0)
    return out
