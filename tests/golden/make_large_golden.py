"""Golden totals / assignments at the benchmarked sizes (TEST INFRASTRUCTURE).

Run in the build container (CPU only; the large cases take tens of minutes to
hours, so each case is its own invocation and writes its own fixture):

    python tests/golden/make_large_golden.py q30 4000 4000 0
    python tests/golden/make_large_golden.py q30 10000 10000 0
    python tests/golden/make_large_golden.py q30 10000 40000 0
    python tests/golden/make_large_golden.py f64 4000 4000 0
    python tests/golden/make_large_golden.py q40 4000 4000 0
    python tests/golden/make_large_golden.py q35 4000 4000 0

Inputs are `paper_2303_13803_b200.synth.make_cluster(n, m, seed)` (the bench's
snapshot generator; pure numpy) and the default table.  W is the oracle's
vectorised `predict_point` restatement (`oracle/predictor_ref.py`, pinned
bit-exact against the reference's own `predict_point` by
tests/test_oracle_golden.py), with the reference's 1e-6 edge rule
(`/root/reference/pkg/src/muxsim/matching.py:19,164-166`).

  q30  -- Wq = rint(W * 2^30) (the bench's quantisation), solved by
          scipy.optimize.linear_sum_assignment(maximize=True) on Wq as float64
          (every partial sum < 2^53, so LSA's arithmetic is exact).  Records the
          optimal integer total.  LSA is independent of this repo's solvers; on
          dyadic weights its totals equal the reference's `max_weight_matching`
          (xcheck.py).
  q35/q40 -- the same with 35- / 40-bit int64 weights, solved by the oracle's
          int64 Hungarian (oracle/hungarian.c, restating matching.py:45-101);
          records its assignment and whether the integer optimum is unique.
  f64  -- the reference algorithm itself on the float64 W: the oracle's C
          restatement of `_solve_min_assignment` (bit-identical col_of_row /
          duals to the reference, pinned on golden duals) on the reference's
          square padding + cost = max - W (matching.py:156-170).  Records the
          reference assignment, its float total, and whether the optimum is
          unique (SCC certificate on the tight-edge digraph).
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def weights(n, m, seed, chunk=1000):
    from oracle import predictor_ref as pr
    from paper_2303_13803_b200.synth import make_cluster
    cl = make_cluster(n, m, seed=seed)
    vals = pr.default_table_values()
    W = np.empty((n, m), dtype=np.float64)
    for r in range(0, n, chunk):
        W[r:r + chunk] = pr.predict_pairs_exact(pr.DEFAULT_AXES, vals, cl.x[r:r + chunk],
                                                cl.share[r:r + chunk], cl.y)
    W[W < 1e-6] = 0.0          # matching.py:19 / 164-166 edge rule
    return W


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    mode, n, m, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    t0 = time.time()
    W = weights(n, m, seed)
    out = {"mode": mode, "n": n, "m": m, "seed": seed,
           "inputs": "paper_2303_13803_b200.synth.make_cluster(n, m, seed), default table",
           "w_sha256": sha(W)}
    if mode in ("q30", "q20"):
        q = int(mode[1:])
        from scipy.optimize import linear_sum_assignment
        Q = np.rint(W * float(2 ** q))
        t1 = time.time()
        r, c = linear_sum_assignment(Q, maximize=True)
        out.update(qbits=q, solver="scipy.optimize.linear_sum_assignment(maximize=True)",
                   total_q=int(Q[r, c].sum()), total_f64_of_lsa=float(W[r, c].sum()),
                   solve_s=time.time() - t1)
    elif mode in ("q35", "q36", "q40"):
        from oracle import matching_ref as mr
        q = int(mode[1:])
        Q = np.rint(W * float(2 ** q)).astype(np.int64)
        nn = max(n, m)
        P = np.zeros((nn, nn), dtype=np.int64)
        P[:n, :m] = Q
        cost = P.max() - P
        t1 = time.time()
        col, u, v = mr.solve_min_assignment(cost)
        solve_s = time.time() - t1
        total = int(P[np.arange(nn), col].sum())
        uniq = bool(mr.is_unique_optimum(cost, col, u, v))
        colr = [int(j) if j < m and Q[i, j] > 0 else -1 for i, j in enumerate(col[:n])]
        out.update(qbits=q, solver="oracle int64 Hungarian (matching.py:45-101 restated)",
                   total_q=total, col_of_row=colr, unique_optimum=uniq, solve_s=solve_s)
    elif mode == "f64":
        from oracle import matching_ref as mr
        nn = max(n, m)
        P = np.zeros((nn, nn))
        P[:n, :m] = W
        cost = P.max() - P
        t1 = time.time()
        col, u, v = mr.solve_min_assignment(cost)
        solve_s = time.time() - t1
        uniq = bool(mr.is_unique_optimum(cost, col, u, v))
        colr = [int(j) if j < m and W[i, j] > 0.0 else -1 for i, j in enumerate(col[:n])]
        tot = 0.0
        for i, j in enumerate(colr):
            if j >= 0:
                tot += float(W[i, j])
        out.update(solver="oracle C restatement of matching._solve_min_assignment on float64 cost",
                   col_of_row=colr, total_f64=tot, unique_optimum=uniq, solve_s=solve_s)
    else:
        raise SystemExit(f"unknown mode {mode}")
    out["wall_s"] = time.time() - t0
    path = os.path.join(HERE, f"large_{mode}_{n}x{m}_s{seed}.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(path, {k: v for k, v in out.items() if k != "col_of_row"})


if __name__ == "__main__":
    main()
