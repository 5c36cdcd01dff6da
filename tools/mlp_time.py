"""Time the MLP plugin on n x m pairs (CUDA events): python tools/mlp_time.py [n] [m]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2303_13803_b200.mlp import MlpPredictor, predict_pairs_mlp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
rng = np.random.default_rng(0)
on = torch.as_tensor(np.stack([rng.uniform(0.2, 1, n), rng.uniform(0.15, 0.8, n), np.full(n, 0.5), rng.uniform(0.01, 0.04, n)], 1), device="cuda")
off = torch.as_tensor(np.stack([rng.uniform(0.6, 1, m), rng.uniform(0.6, 0.98, m), np.full(m, 0.5), np.full(m, 0.1)], 1), device="cuda")
share = torch.as_tensor(np.floor(rng.uniform(0.15, 0.8, n) / 0.05 + 1e-6) * 0.05, device="cuda")
mlp = MlpPredictor.random(0)
out = torch.empty((n, (m + 3) // 4 * 4), dtype=torch.float32, device="cuda")
for _ in range(3):
    predict_pairs_mlp(mlp, on, share, off, out=out)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); predict_pairs_mlp(mlp, on, share, off, out=out); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[5]
fl = (2.0 * 64 * 64 * 2 + 4.0 * 64) * n * m
print(f"mlp {n}x{m}: {ms:.3f} ms, {fl / ms / 1e9:.1f} TFLOP/s algorithmic, {2.0 * (144 + 128) * 64 * n * m / ms / 1e9:.1f} issued")
