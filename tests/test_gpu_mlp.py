"""MLP plugin (tcgen05 kernel) against its float64 oracle.  Parity is
UNPINNED relative to the reference (which has no MLP); the oracle is
oracle/mlp_ref.py on the same weights.

Two checks: (1) against a numpy emulation of the kernel's precision (bf16
rounding of the layer-1/2 activations and of W2/W3, fp32 elsewhere) -- this
pins the tensor-core data path to 1e-4; (2) against the pure float64 network
-- this measures what bf16 operands cost (documented bound: 2e-2 absolute on
outputs in [0, 1])."""

import numpy as np
import pytest

from oracle import mlp_ref

pytestmark = pytest.mark.gpu


def bf16(x):
    x = np.asarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def emulated(params, on, share, off):
    """Kernel-precision forward: P/Q fp32, h1/W2/h2/W3 and the layer-2/3
    biases bf16 (they ride in the GEMM as a ones column), fp32 accumulate."""
    f32 = np.float32
    W1 = params["W1"].astype(f32)
    shift, scale = params["shift"].astype(f32), params["scale"].astype(f32)
    x_on = ((on - shift[:4].astype(np.float64)) * scale[:4].astype(np.float64)).astype(f32)
    x_off = ((off - shift[4:8].astype(np.float64)) * scale[4:8].astype(np.float64)).astype(f32)
    x_s = ((share - float(shift[8])) * float(scale[8])).astype(f32)
    P = x_on @ W1[:, :4].T + x_s[:, None] * W1[:, 8][None, :] + params["b1"].astype(f32)
    Q = x_off @ W1[:, 4:8].T
    W2, W3 = bf16(params["W2"]), bf16(params["W3"])
    out = np.empty((P.shape[0], Q.shape[0]), dtype=np.float64)
    for u in range(P.shape[0]):
        h1 = bf16(np.maximum(P[u][None, :] + Q, 0))
        h2 = bf16(np.maximum(h1 @ W2.T + bf16(params["b2"]), 0))
        h3 = np.maximum(h2 @ W3.T + bf16(params["b3"]), 0)
        out[u] = np.clip(h3 @ params["w4"].astype(f32) + f32(params["b4"]), 0, 1)
    return out


def _inputs(n, m, seed):
    rng = np.random.default_rng(seed)
    on = np.stack([rng.uniform(0.2, 1.0, n), rng.uniform(0.15, 0.8, n), np.full(n, 0.5),
                   rng.uniform(0.01, 0.04, n)], axis=1)
    off = np.stack([rng.uniform(0.6, 1.0, m), rng.uniform(0.6, 0.98, m), np.full(m, 0.5),
                    np.full(m, 0.1)], axis=1)
    share = np.floor(rng.uniform(0.15, 0.8, n) / 0.05 + 1e-6) * 0.05
    return on, share, off


@pytest.mark.parametrize("n,m,seed", [(1, 1, 0), (3, 129, 1), (130, 300, 2), (257, 1000, 3)])
def test_mlp_kernel_matches_emulation(cuda, n, m, seed):
    from paper_2303_13803_b200.mlp import MlpPredictor, predict_pairs_mlp
    mlp = MlpPredictor.random(seed)
    on, share, off = _inputs(n, m, seed)
    W = predict_pairs_mlp(mlp, on, share, off).cpu().numpy().astype(np.float64)
    E = emulated(mlp.params(), on, share, off)
    d = np.abs(W - E)
    # fp32 accumulation order can flip one bf16 rounding of an activation:
    # nearly every entry agrees to fp32 precision, a few move by ~1 bf16 ulp
    assert np.quantile(d, 0.99) < 1e-5
    assert d.max() < 5e-3


def test_mlp_kernel_vs_float64(cuda):
    from paper_2303_13803_b200.mlp import MlpPredictor, predict_pairs_mlp
    mlp = MlpPredictor.random(7)
    on, share, off = _inputs(200, 700, 7)
    W = predict_pairs_mlp(mlp, on, share, off).cpu().numpy().astype(np.float64)
    R = mlp_ref.forward(mlp.params(), on, share, off)
    assert 0.05 < R.mean() < 0.95          # the random net spans (0, 1)
    assert np.max(np.abs(W - R)) < 2e-2


def test_mlp_quantised_output_and_matching(cuda):
    import torch
    from paper_2303_13803_b200 import match_dense
    from paper_2303_13803_b200.mlp import MlpPredictor, predict_pairs_mlp
    from oracle import matching_ref
    mlp = MlpPredictor.random(3)
    on, share, off = _inputs(300, 280, 3)
    Wf = predict_pairs_mlp(mlp, on, share, off).cpu().numpy().astype(np.float64)
    Q = predict_pairs_mlp(mlp, on, share, off, dtype="int32", qbits=20)
    Qh = Q.cpu().numpy().astype(np.int64)
    want = np.rint(np.where(Wf >= 1e-6, Wf, 0) * 2.0 ** 20).astype(np.int64)
    assert np.array_equal(Qh, want)
    full = torch.zeros((300, 280), dtype=torch.int32, device="cuda")
    full.copy_(Q)
    col, total = match_dense(full)
    opt, _ = matching_ref.max_weight_total_int(Qh)
    assert total == opt
