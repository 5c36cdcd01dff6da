"""Config-5 replay fixture from the REFERENCE trace generator (TEST INFRASTRUCTURE).

Run in the build container (imports /root/reference/pkg/src read-only):
    python tests/golden/make_replay_fixture.py            # the fixture
    python tests/golden/make_replay_fixture.py --totals   # LSA totals of sampled rounds

BASELINE.json config 5: "rectangular 10k online x 40k offline candidates,
100-round trace replay with dynamic SM-share features".  The trace is
`muxsim.gen.gen_trace({"gpus": 10000, "horizon_s": 90000,
"offline": {"count_per_gpu": 4.0}}, seed=0)` (gen.py:67-167).  Round k runs at
t = k * 900 s (SchedulerConfig.interval); its rows are the 10k onlines with
the reference's own `peak_online_profile` / `dynamic_sm` (scheduler.py:99-135)
at t, its columns every offline job submitted by t.

Stored compactly (npz): per online its 8 profile SM levels (float64) and per
round the index of the peak level (uint8) and the share in quanta (uint8,
share = k * 0.05, bit-identical to quantize_share's floor(.) * quantum);
per offline job its SM demand, memory fraction and submit time.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main(rounds=100, seed=0):
    sys.path.insert(0, REF)
    from muxsim.gen import gen_trace
    from muxsim.scheduler import SchedulerConfig, dynamic_sm, peak_online_profile
    spec = {"gpus": 10000, "horizon_s": 90000, "offline": {"count_per_gpu": 4.0}}
    tr = gen_trace(spec, seed=seed)
    cfg = SchedulerConfig()
    n = len(tr.online)
    levels = np.array([[p.sm_activity for _q, p in w.profile_by_qps] for w in tr.online])
    lvl = np.zeros((rounds, n), dtype=np.uint8)
    shq = np.zeros((rounds, n), dtype=np.uint8)
    for k in range(rounds):
        t = (k + 1) * cfg.interval
        for u, w in enumerate(tr.online):
            pk = peak_online_profile(w, t - cfg.interval, t).sm_activity
            lvl[k, u] = int(np.nonzero(levels[u] == pk)[0][0])
            s = dynamic_sm(w, t, cfg)
            q = int(round(s / cfg.quantum))
            assert q * cfg.quantum == s, (s, q)
            shq[k, u] = q
    y = np.array([v.profile.sm_activity for v in tr.offline])
    mem = np.array([v.profile.mem_fraction for v in tr.offline])
    sub = np.array([v.submit_time for v in tr.offline])
    out = os.path.join(HERE, "replay_cfg5.npz")
    np.savez_compressed(out, levels=levels, lvl=lvl, share_q=shq, y=y, mem=mem, submit=sub,
                        interval=cfg.interval, quantum=cfg.quantum, spec=str(spec), seed=seed)
    print(out, os.path.getsize(out), "bytes;", n, "onlines,", len(y), "offline jobs")




def round_arrays_np(fx, k):
    """Rows / columns of replay round k from the fixture (same rule as
    paper_2303_13803_b200.replay)."""
    n = fx["levels"].shape[0]
    x = fx["levels"][np.arange(n), fx["lvl"][k]]
    share = fx["share_q"][k].astype(np.float64) * float(fx["quantum"])
    rows = np.nonzero(share > 0.0)[0]
    t = (k + 1) * float(fx["interval"])
    cols = np.nonzero((fx["submit"] <= t) & (fx["mem"] <= 0.40))[0]
    return x[rows], share[rows], fx["y"][cols]


def totals(ks=(0, 1, 2, 5), qbits=30):
    """scipy LSA optimal totals of sampled replay rounds (quantised weights)."""
    import json
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from scipy.optimize import linear_sum_assignment
    from oracle import predictor_ref as pr
    fx = np.load(os.path.join(HERE, "replay_cfg5.npz"))
    vals = pr.default_table_values()
    out = {}
    for k in ks:
        x, s, y = round_arrays_np(fx, k)
        W = pr.predict_pairs_exact(pr.DEFAULT_AXES, vals, x, s, y)
        W[W < 1e-6] = 0.0
        Q = np.rint(W * float(2 ** qbits))
        r, c = linear_sum_assignment(Q, maximize=True)
        out[str(k)] = {"n": int(x.size), "m": int(y.size), "total_q": int(Q[r, c].sum())}
        print(k, out[str(k)], flush=True)
    with open(os.path.join(HERE, "replay_cfg5_totals.json"), "w") as f:
        json.dump({"qbits": qbits, "solver": "scipy.optimize.linear_sum_assignment(maximize=True)",
                   "rounds": out}, f)


if __name__ == "__main__":
    if "--totals" in sys.argv:
        totals()
    else:
        main()
