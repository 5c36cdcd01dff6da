"""One 1200 x 1200 predictor solve (used to probe solver variants by env)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2303_13803_b200 import _native as nat, default_table
from paper_2303_13803_b200.synth import make_cluster
from oracle import predictor_ref as pr
n = int(os.environ.get("N", "1200")); seed = int(os.environ.get("SEED", "30"))
cl = make_cluster(n, n, seed=seed)
t = default_table()
W = pr.predict_pairs_exact(t.axes, t.values, cl.x, cl.share, cl.y)
Q = np.rint(np.where(W >= 1e-6, W, 0.0) * 2.0 ** 30).astype(np.int32)
ldw = (n + 3) // 4 * 4
P = np.zeros((n, ldw), np.int32); P[:, :n] = Q
Wq = torch.as_tensor(P, device="cuda")
rk = torch.as_tensor(cl.x, device="cuda"); ck = torch.as_tensor(cl.y, device="cuda")
col = torch.empty(n, dtype=torch.int32, device="cuda")
tot, st = nat.ctypes.c_int64(0), nat.MuxStats()
nat.check(nat.load().mux_match_keyed(nat.context(0), Wq.data_ptr(), nat.MUX_W_I32, n, n, ldw, rk.data_ptr(), ck.data_ptr(),
                                     col.data_ptr(), 0, nat.ctypes.byref(tot), nat.ctypes.byref(st), nat.stream_ptr()))
print("total", tot.value)
