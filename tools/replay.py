"""Config 5 of BASELINE.json: a 100-round trace replay on one B200.

10k online workloads whose peak SM activity drifts from round to round (the
offered share is recomputed with the reference's dynamic_sm formula each
round), and an offline job set that grows as jobs are submitted: round k
sees the first min(40000, 400 (k + 1)) jobs (the column set is
"submitted-by-t", growing to 40k).  Early rounds have fewer jobs than online
rows (N > M, transposed solve), round 24 is square, later rounds are
rectangular N < M.  Every round goes through the C ABI `mux_round` with host
arrays (H2D features, exact scoring, exact matching, canonicalisation, D2H).
Prints one JSON line with per-round times and totals.
"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_13803_b200 import default_table
from paper_2303_13803_b200.scheduler import round_arrays
from paper_2303_13803_b200.synth import shares_for

rounds = int(os.environ.get("ROUNDS", "100"))
N, MMAX, STEP, q = 10000, 40000, 400, int(os.environ.get("QBITS", "30"))
rng = np.random.default_rng(0)
base = rng.uniform(0.15, 0.80, N)
phase = rng.uniform(0, 2 * np.pi, N)
y_all = rng.uniform(0.60, 0.98, MMAX)
t = default_table()
round_arrays(t, base, shares_for(base), y_all, qbits=q)   # warm-up at the largest size (workspace allocations)
rows = []
t_all = time.perf_counter()
for k in range(rounds):
    x = np.clip(base + 0.05 * np.sin(phase + 0.3 * k), 0.0, 1.0)
    s = shares_for(x)
    keep = s > 0
    xs, ss = x[keep], s[keep]
    m = min(MMAX, STEP * (k + 1))
    t0 = time.perf_counter()
    col, total, st = round_arrays(t, xs, ss, y_all[:m], qbits=q, stats=True)
    ms = (time.perf_counter() - t0) * 1e3
    rows.append({"round": k, "n": int(xs.shape[0]), "m": m, "ms": ms, "total_q": total,
                 "placed": int((col >= 0).sum()), "ms_match": st["ms_match"]})
    print(f"round {k:3d} n {xs.shape[0]} m {m:5d}: {ms:8.1f} ms  placed {rows[-1]['placed']}", file=sys.stderr, flush=True)
wall = time.perf_counter() - t_all
ms_list = [r["ms"] for r in rows]
print(json.dumps({"config": "100-round replay, 10k online x growing offline set (to 40k), q=%d" % q,
                  "rounds": rounds, "wall_s": wall, "ms_per_round_mean": float(np.mean(ms_list)),
                  "ms_per_round_median": float(np.median(ms_list)), "ms_per_round_max": float(np.max(ms_list)),
                  "per_round": rows}))
