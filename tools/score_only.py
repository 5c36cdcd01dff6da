"""Scoring-only driver for profiling K1 (`score_exact_kernel`): one 10k x 10k
exact-mode table scoring into int32 weights at q = 30, timed with CUDA events
after warm-up.  Usage: python tools/score_only.py [N] [M]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_13803_b200 import predictor, tables  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
rng = np.random.default_rng(0)
x = torch.as_tensor(rng.uniform(0.15, 0.80, n), device="cuda")
s = torch.as_tensor(np.floor((1.0 - x.cpu().numpy() - 0.05) / 0.05 + 1e-6) * 0.05, device="cuda")
y = torch.as_tensor(rng.uniform(0.60, 0.98, m), device="cuda")
t = tables.default_table()
out = predictor.predict_pairs(t, x, s, y, dtype="int32", qbits=30)
for _ in range(3):
    predictor.predict_pairs(t, x, s, y, dtype="int32", qbits=30, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
reps = 10
for _ in range(reps):
    predictor.predict_pairs(t, x, s, y, dtype="int32", qbits=30, out=out)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
gbs = 4.0 * n * m / (ms * 1e-3) / 1e9
print(f"score_exact {n}x{m}: {ms:.4f} ms/launch (incl. host call), {gbs:.1f} GB/s algorithmic write")
