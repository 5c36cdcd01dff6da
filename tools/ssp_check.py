"""GPU check of the multilevel shortest-path solver (csrc/ssp.cu): totals vs
scipy / the oracle Hungarian, the dense dual certificate at every level
(MUX_SSP_CHECK=1), and timings at 10k."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MUX_SSP_CHECK", "1")
import torch
from scipy.optimize import linear_sum_assignment
from paper_2303_13803_b200 import default_table
from paper_2303_13803_b200.scheduler import round_arrays
from paper_2303_13803_b200.matching import match_dense
from paper_2303_13803_b200.synth import make_cluster
from oracle import predictor_ref as pr

t = default_table()
fails = 0
def lsa_total(Q):
    r, c = linear_sum_assignment(Q.astype(np.float64), maximize=True)
    return int(Q[r, c].sum())

cases = [(64, 20, 0), (200, 20, 1), (500, 30, 2), (1000, 20, 3), (1000, 30, 4), (1500, 30, 5)]
for n, q, seed in cases:
    cl = make_cluster(n, n, seed=seed)
    W = pr.predict_pairs_exact(pr.DEFAULT_AXES, pr.default_table_values(), cl.x, cl.share, cl.y)
    Q = np.rint(np.where(W >= 1e-6, W, 0) * 2.0 ** q).astype(np.int64)
    want = lsa_total(Q)
    col, tot, st = round_arrays(t, cl.x, cl.share, cl.y, qbits=q, stats=True)
    ok = tot == want and int(Q[np.arange(n)[col >= 0], col[col >= 0]].sum()) == want
    Qt = torch.tensor(Q.astype(np.int32), device="cuda")
    col2, tot2 = match_dense(Qt)
    ok2 = tot2 == want
    fails += (not ok) + (not ok2)
    print(f"n={n} q={q}: round {tot} match {tot2} want {want} {'OK' if ok and ok2 else 'FAIL'} ms {st['ms_match']:.2f}", flush=True)
# random uniform matrices (generic keys)
for n, hi, seed in [(300, 1000, 0), (1000, 1 << 20, 1), (777, 50, 2)]:
    rng = np.random.default_rng(seed)
    Q = rng.integers(1, hi, (n, n)).astype(np.int64)
    want = lsa_total(Q)
    ldw = (n + 3) // 4 * 4
    Qp = np.zeros((n, ldw), np.int32); Qp[:, :n] = Q
    col2, tot2 = match_dense(torch.tensor(Qp, device="cuda"), n, n)
    fails += tot2 != want
    print(f"random n={n} hi={hi}: {tot2} want {want} {'OK' if tot2 == want else 'FAIL'}", flush=True)
# large: certificate only + timing
for n, q in [(4000, 30), (10000, 30), (10000, 20)][: int(os.environ.get('NBIG', '3'))]:
    cl = make_cluster(n, n, seed=0)
    for rep in range(2):
        t0 = time.time()
        col, tot, st = round_arrays(t, cl.x, cl.share, cl.y, qbits=q, stats=True)
        print(f"n={n} q={q} rep {rep}: total {tot} ms_match {st['ms_match']:.2f} wall {1e3*(time.time()-t0):.1f} ms", flush=True)
print("FAILS", fails)
