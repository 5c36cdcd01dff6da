"""Int64-weight solver smoke cases (one per process, under an outer timeout)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2303_13803_b200 import _native as nat
n, m, hi, seed = (int(a) for a in sys.argv[1:5])
Q = np.random.default_rng(seed).integers(1, hi, size=(n, m)).astype(np.int64)
ldw = max(2, (m + 1) // 2 * 2)
P = np.zeros((n, ldw), dtype=np.int64); P[:, :m] = Q
Wq = torch.as_tensor(P, device="cuda")
col = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
tot, st = nat.ctypes.c_int64(0), nat.MuxStats()
rc = nat.load().mux_match_keyed(nat.context(0), Wq.data_ptr(), nat.MUX_W_I64, n, m, ldw, None, None, col.data_ptr(), 0,
                                nat.ctypes.byref(tot), nat.ctypes.byref(st), nat.stream_ptr())
torch.cuda.synchronize()
from scipy.optimize import linear_sum_assignment
r, c = linear_sum_assignment(Q.astype(np.float64), maximize=True)
print(n, m, hi, "rc", rc, nat.load().mux_last_error().decode() if rc else "", "total", tot.value, "lsa", int(Q[r, c].sum()), flush=True)
