"""Rectangular (N < M) rounds on the multilevel solver: totals vs scipy LSA
(rectangular) with the dual certificate, then the 4k x 12k / 10k x 40k
configs against the auction's totals from profiles/r01."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MUX_SSP_CHECK", "1")
from scipy.optimize import linear_sum_assignment
from paper_2303_13803_b200 import default_table
from paper_2303_13803_b200.scheduler import round_arrays
from paper_2303_13803_b200.synth import make_cluster
from oracle import predictor_ref as pr
t = default_table()
fails = 0
for n, m, q, seed in [(50, 64, 20, 0), (300, 900, 20, 1), (1000, 3000, 30, 2), (999, 1001, 30, 3), (1500, 6000, 20, 4), (64, 50, 20, 5), (3000, 1000, 30, 6), (1001, 999, 20, 7)]:
    cl = make_cluster(n, m, seed=seed)
    W = pr.predict_pairs_exact(pr.DEFAULT_AXES, pr.default_table_values(), cl.x, cl.share, cl.y)
    Q = np.rint(np.where(W >= 1e-6, W, 0) * 2.0 ** q).astype(np.int64)
    r, c = linear_sum_assignment(Q.astype(np.float64), maximize=True)
    want = int(Q[r, c].sum())
    t0 = time.time()
    col, tot, st = round_arrays(t, cl.x, cl.share, cl.y, qbits=q, stats=True)
    ok = tot == want and int(Q[np.arange(n)[col >= 0], col[col >= 0]].sum()) == want and len(set(col[col >= 0].tolist())) == (col >= 0).sum()
    fails += not ok
    print(f"{n}x{m} q={q}: {tot} want {want} {'OK' if ok else 'FAIL'} ({1e3*(time.time()-t0):.1f} ms, match {st['ms_match']:.1f})", flush=True)
os.environ["MUX_SSP_CHECK"] = "0"
for n, m, q, want in [(4000, 12000, 20, 2413913397), (12000, 4000, 20, 3042374446), (10000, 40000, 20, 6111445217), (10000, 40000, 30, None)]:
    cl = make_cluster(n, m, seed=0)
    for rep in range(2):
        t0 = time.time()
        col, tot, st = round_arrays(t, cl.x, cl.share, cl.y, qbits=q, stats=True)
        ok = want is None or tot == want
        fails += not ok
        print(f"{n}x{m} q={q} rep {rep}: {tot} want {want} {'OK' if ok else 'FAIL'} wall {1e3*(time.time()-t0):.1f} ms match {st['ms_match']:.1f} dense {st['ms_dense']:.1f} ({st['dense_steps']} pops, {st['dense_searches']} searches) par {st['ms_parallel']:.1f}", flush=True)
print("FAILS", fails)
