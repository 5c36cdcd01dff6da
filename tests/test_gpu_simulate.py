"""The reference's simulator driven by the GPU round.

The unmodified reference package (baseline/_ref, pip-installed from the
reference; loaded under its own name so it cannot collide with this repo's
`muxsim` shim) runs its event engine (`simengine.run`, the per-round caller
`_Engine._on_round`, simengine.py:665-735) over its own bundled trace suite
with `simengine.schedule` replaced by this repo's GPU `schedule()`:

* every round the engine schedules is also scheduled by the reference's own
  `schedule()`; both placements have the same float64 total within config
  3's tolerance (rounds whose pairs differ are ties or near-ties at the
  40-bit quantisation; their count and gap are reported);
* the paper's acceptance criteria 5 and 6 (test_acceptance.py:108-144:
  online latency vs solo, throughput vs the time-sharing / fixed-share /
  random-match baselines) hold with the GPU round in the loop.
"""

import importlib
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref", "muxsim")
POLICIES = ("muxflow", "online_only", "pb_time_sharing", "muxflow_fixed_sm", "muxflow_random_match")


@pytest.fixture(scope="module")
def ref():
    """The reference package's modules, imported as `muxsim` from baseline/_ref
    with any other `muxsim` (this repo's shim) set aside for the import and
    restored afterwards (the reference has no function-level imports, so its
    modules keep their own references)."""
    base = os.path.dirname(REF)
    assert os.path.isfile(os.path.join(REF, "__init__.py")), \
        "reference package missing: pip install --no-index --target baseline/_ref <reference>/pkg"
    saved = {k: v for k, v in sys.modules.items() if k == "muxsim" or k.startswith("muxsim.")}
    for k in saved:
        del sys.modules[k]
    sys.path.insert(0, base)
    try:
        mods = {k: importlib.import_module(f"muxsim.{k}") for k in ("simengine", "suite", "scheduler", "predictor")}
        assert all(os.path.abspath(m.__file__).startswith(os.path.abspath(base)) for m in mods.values())
    finally:
        sys.path.remove(base)
        for k in [k for k in sys.modules if k == "muxsim" or k.startswith("muxsim.")]:
            del sys.modules[k]
        sys.modules.update(saved)
    return mods


def _run(ref, trace, seed, policy, gpu):
    from paper_2303_13803_b200 import schedule as gpu_schedule
    se = ref["simengine"]
    cfg = se.SimConfig(scheduler=ref["scheduler"].SchedulerConfig(policy=policy))
    saved = se.schedule
    try:
        if gpu:
            se.schedule = gpu_schedule
        return se.run(trace, cfg, seed=seed)
    finally:
        se.schedule = saved


def test_every_simulated_round_matches_the_reference_schedule(cuda, ref):
    """Each round the reference engine schedules (its own snapshots, in its
    own order) is scheduled by both: the placements must have the same
    float64 total (predict over the reference table) -- the rounds whose
    pairs differ are ties or near-ties at the 40-bit quantisation, reported."""
    from paper_2303_13803_b200 import schedule as gpu_schedule
    se, sc = ref["simengine"], ref["scheduler"]
    pr = ref["predictor"]
    stock_schedule = se.schedule
    stats = {"rounds": 0, "differ": 0, "max_gap": 0.0}

    def both(online, offline, states, table, cfg, now, rng=None):
        import copy
        a = stock_schedule(online, offline, states, table, cfg, now, rng=copy.deepcopy(rng))
        b = gpu_schedule(online, offline, states, table, cfg, now, rng=rng)
        stats["rounds"] += 1
        if a.pairs != b.pairs:
            stats["differ"] += 1
            by_id = {u.id: u for u in online}
            off = {v.id: v for v in offline}

            def total(asg):
                t = 0.0
                for _g, uid, vid, sm in asg.pairs:
                    peak = sc.peak_online_profile(by_id[uid], now - cfg.interval, now)
                    t += pr.predict(table, peak, off[vid].profile, sm)
                return t
            gap = total(a) - total(b)
            stats["max_gap"] = max(stats["max_gap"], abs(gap))
            assert abs(gap) <= len(online) * 2.0 ** -20, gap
        return b

    for name, trace, seed in ref["suite"].suite_traces()[:3]:
        cfg = se.SimConfig(scheduler=sc.SchedulerConfig(policy="muxflow"))
        saved = se.schedule
        try:
            se.schedule = both
            se.run(trace, cfg, seed=seed)
        finally:
            se.schedule = saved
    assert stats["rounds"] > 0
    print(f"simulated rounds {stats['rounds']}, placements differ in {stats['differ']}, "
          f"max float64 total gap {stats['max_gap']:.3e}")


def test_acceptance_criteria_5_and_6_with_the_gpu_round(cuda, ref):
    runs = {}
    for name, trace, seed in ref["suite"].suite_traces():
        runs[name] = {p: _run(ref, trace, seed, p, gpu=True) for p in POLICIES}
    # criterion 5 (test_acceptance.py:108-120): online latency safe versus solo
    for name, per in runs.items():
        mux, solo = per["muxflow"], per["online_only"]
        for wid in mux.avg_latency_s:
            assert mux.avg_latency_s[wid] / solo.avg_latency_s[wid] <= 1.20, (name, wid)
            assert mux.p99_latency_s[wid] / solo.p99_latency_s[wid] <= 1.25, (name, wid)
    # criterion 6 (test_acceptance.py:123-144): throughput beats the baselines
    strict = [0, 0, 0]
    for name, per in runs.items():
        mux, pb, fixed, rnd = (per[p] for p in ("muxflow", "pb_time_sharing", "muxflow_fixed_sm",
                                                "muxflow_random_match"))
        assert mux.avg_jct_s <= pb.avg_jct_s, name
        assert mux.oversold_gpu >= fixed.oversold_gpu, name
        assert mux.oversold_gpu >= rnd.oversold_gpu, name
        strict[0] += mux.avg_jct_s < pb.avg_jct_s
        strict[1] += mux.oversold_gpu > fixed.oversold_gpu
        strict[2] += mux.oversold_gpu > rnd.oversold_gpu
    assert strict[0] >= 4 and strict[1] >= 4 and strict[2] >= 4, strict
