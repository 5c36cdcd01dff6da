"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports the reference `muxsim` read-only from /root/reference/pkg/src and
writes small JSON fixtures next to this script.  The fixtures are committed;
the GPU box never needs /root/reference.  Each fixture records which
reference function produced it.
"""

import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    sys.path.insert(0, REF)
    sys.path.insert(1, ROOT)
    from muxsim import core as rcore
    from muxsim import gpu_state as rgpu
    from muxsim.matching import BipartiteGraph, _solve_min_assignment, max_weight_matching
    from muxsim.predictor import build_table_from_model, predict_point
    from muxsim.scheduler import SchedulerConfig, dynamic_sm, schedule
    from muxsim.simengine import SimConfig, default_table

    class _CoreShim:   # records from the reference's own modules
        WorkloadProfile = rcore.WorkloadProfile
        OnlineWorkload = rcore.OnlineWorkload
        OfflineWorkload = rcore.OfflineWorkload
        HealthState = rgpu.HealthState

    from paper_2303_13803_b200.synth import make_cluster, records

    out = {}
    # --- predictor (predictor.py:85-112) on the default table (simengine.py:197-203)
    t = default_table(SimConfig())
    rng = random.Random(2303)
    pts = [(0.0, 0.5, 0.0), (1.0, 1.0, 1.0), (0.5, 0.2, 0.5), (0.125, 0.5625, 1 / 9),
           (0.3, 0.75, 0.45), (0.999999, 0.6, 0.05), (0.5, 0.75, 1.0)]
    for _ in range(2000):
        pts.append((rng.random(), rng.uniform(0.3, 1.0), rng.random()))
    out["predict_default"] = {
        "source": "muxsim.predictor.predict_point(default_table(SimConfig()), x, y, z)",
        "axes": [list(t.online_sm), list(t.offline_sm), list(t.sm_pct)],
        "values": [float(v) for v in t.values.reshape(-1)],
        "points": [[x, y, z, predict_point(t, x, y, z)] for x, y, z in pts],
    }
    # linear-model table (tests/test_predictor.py:24-43)
    axes = (tuple(i / 8 for i in range(9)), tuple(0.5 + i / 16 for i in range(9)),
            tuple(i / 9 for i in range(10)))
    lin = build_table_from_model(lambda x, y, z: 0.1 + 0.2 * x + 0.25 * y + 0.4 * z, *axes)
    lpts = [(rng.random(), rng.uniform(0.5, 1.0), rng.random()) for _ in range(300)]
    out["predict_linear"] = {
        "source": "predict_point on build_table_from_model(linear_model, AXES)",
        "axes": [list(a) for a in axes],
        "values": [float(v) for v in lin.values.reshape(-1)],
        "points": [[x, y, z, predict_point(lin, x, y, z)] for x, y, z in lpts],
    }

    # --- matching (matching.py:148-208) on dyadic random graphs
    def rgraph(r, max_side, gran):
        nl, nr = r.randint(0, max_side), r.randint(0, max_side)
        L = tuple(f"l{i:02d}" for i in range(nl))
        R = tuple(f"r{j:02d}" for j in range(nr))
        w = {}
        for l in L:
            for rr in R:
                if r.random() < 0.7:
                    w[(l, rr)] = r.randrange(gran + 1) / gran
        return L, R, w

    cases = []
    r = random.Random(1337)
    for trial in range(300):
        L, R, w = rgraph(r, 6 if trial < 200 else 24, 64)
        m = max_weight_matching(BipartiteGraph(L, R, w))
        cases.append({"left": list(L), "right": list(R),
                      "edges": [[a, b, x] for (a, b), x in sorted(w.items())],
                      "pairs": [list(p) for p in m.pairs], "total": m.total_weight})
    # fixed examples: Fig. 7 (test_matching.py:64-72), ties (test_matching.py:106-113)
    for L, R, w in ((("A", "B"), ("C", "D", "E"),
                     {("A", "C"): 0.3, ("A", "D"): 0.8, ("B", "C"): 0.8, ("B", "E"): 0.4}),
                    (("a", "b"), ("x", "y"),
                     {("a", "x"): 0.5, ("a", "y"): 0.5, ("b", "x"): 0.5, ("b", "y"): 0.5})):
        m = max_weight_matching(BipartiteGraph(L, R, w))
        cases.append({"left": list(L), "right": list(R),
                      "edges": [[a, b, x] for (a, b), x in sorted(w.items())],
                      "pairs": [list(p) for p in m.pairs], "total": m.total_weight})
    out["matching"] = {"source": "muxsim.matching.max_weight_matching", "cases": cases}

    # --- Hungarian duals (matching.py:45-101)
    hr = np.random.default_rng(5)
    hung = []
    for n in (1, 2, 5, 17, 40):
        c = np.floor(hr.random((n, n)) * 256) / 256
        col, u, v = _solve_min_assignment(c)
        hung.append({"cost": c.tolist(), "col": col.tolist(), "u": u.tolist(), "v": v.tolist()})
    out["hungarian"] = {"source": "muxsim.matching._solve_min_assignment", "cases": hung}

    # --- dynamic_sm (scheduler.py:123-135) on flat onlines
    cfg = SchedulerConfig()
    flat = []
    sr = random.Random(9)
    for _ in range(300):
        sm = sr.random()
        prof = rcore.WorkloadProfile(sm_activity=sm, gpu_utilization=min(1.0, 1.8 * sm),
                                     sm_occupancy=0.5, iter_time_separate=0.1, mem_fraction=0.3)
        onl = rcore.OnlineWorkload(id="u", gpu_id="g", base_latency=0.02, latency_slo=0.2,
                                   qps_series=((0.0, 100.0),), profile_by_qps=((100.0, prof),))
        flat.append([sm, dynamic_sm(onl, 900.0, cfg)])
    out["dynamic_sm"] = {"source": "muxsim.scheduler.dynamic_sm(flat online, 900, SchedulerConfig())",
                         "cases": flat}

    # --- full rounds (scheduler.py:220-241) on synthetic clusters
    rounds = []
    for (n, m, seed) in ((24, 20, 0), (40, 64, 1), (64, 64, 2), (80, 50, 3), (128, 128, 4)):
        cl = make_cluster(n, m, seed=seed)
        onl, off, states = records(cl, core=_CoreShim)
        asg = schedule(onl, off, states, t, SchedulerConfig(), now=900.0)
        rounds.append({"n": n, "m": m, "seed": seed, "pairs": [list(p) for p in asg.pairs],
                       "unplaced": list(asg.unplaced)})
    out["rounds"] = {"source": "muxsim.scheduler.schedule(records(make_cluster(n, m, seed)), "
                               "default_table, SchedulerConfig(), now=900)", "cases": rounds}

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
