"""Run only the MLP plugin kernel (for ncu): python tools/mlp_only.py N M"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2303_13803_b200.mlp import MlpPredictor, predict_pairs_mlp

n, m = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(0)
on = np.stack([rng.uniform(0.2, 1, n), rng.uniform(0.15, 0.8, n), np.full(n, 0.5), rng.uniform(0.01, 0.04, n)], 1)
off = np.stack([rng.uniform(0.6, 1, m), rng.uniform(0.6, 0.98, m), np.full(m, 0.5), np.full(m, 0.1)], 1)
share = np.floor(rng.uniform(0.15, 0.8, n) / 0.05 + 1e-6) * 0.05
mlp = MlpPredictor.random(0)
for _ in range(3):
    W = predict_pairs_mlp(mlp, on, share, off)
torch.cuda.synchronize()
print("ok", float(W.mean()))
