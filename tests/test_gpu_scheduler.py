"""schedule() through the GPU round: the reference's scheduler tests
(pkg/tests/test_scheduler.py:152-278) and golden rounds from the reference."""

import random
import types

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def prof(sm, mem=0.30):
    from paper_2303_13803_b200 import WorkloadProfile
    return WorkloadProfile(sm_activity=sm, gpu_utilization=min(1.0, 1.8 * sm), sm_occupancy=0.5,
                           iter_time_separate=0.1, mem_fraction=mem)


def flat_online(oid, gpu, sm, mem=0.30):
    from paper_2303_13803_b200 import OnlineWorkload
    return OnlineWorkload(id=oid, gpu_id=gpu, base_latency=0.02, latency_slo=0.2,
                          qps_series=((0.0, 100.0),), profile_by_qps=((100.0, prof(sm, mem)),))


def offline(oid, dem, mem=0.20):
    from paper_2303_13803_b200 import OfflineWorkload
    return OfflineWorkload(id=oid, submit_time=0.0, work_separate=3600.0, profile=prof(dem, mem))


def healthy(*gpus):
    from paper_2303_13803_b200 import HealthState
    return {g: HealthState.HEALTHY for g in gpus}


def crafted_table():
    from paper_2303_13803_b200 import PredictionTable
    values = np.array([[[0.25, 0.30], [0.60, 0.80], [0.20, 0.35]],
                       [[0.80, 0.85], [0.30, 0.30], [0.40, 0.45]]])
    return PredictionTable("default", (0.20, 0.60), (0.25, 0.50, 0.90), (0.35, 0.75), values)


def fixture():
    return ([flat_online("on-A", "g0", 0.20), flat_online("on-B", "g1", 0.60)],
            [offline("off-C", 0.25), offline("off-D", 0.50), offline("off-E", 0.90)])


def test_picks_max_weight_pairing(cuda):
    from paper_2303_13803_b200 import SchedulerConfig, schedule
    onl, offs = fixture()
    asg = schedule(onl, offs, healthy("g0", "g1"), crafted_table(), SchedulerConfig(), now=900.0)
    assert [p[:3] for p in asg.pairs] == [("g0", "on-A", "off-D"), ("g1", "on-B", "off-C")]
    shares = {p[1]: p[3] for p in asg.pairs}
    assert shares["on-A"] == pytest.approx(0.75) and shares["on-B"] == pytest.approx(0.35)
    assert asg.unplaced == ("off-E",)


def test_only_healthy_gpus(cuda):
    from paper_2303_13803_b200 import HealthState, SchedulerConfig, schedule
    onl, offs = fixture()
    st = {"g0": HealthState.UNHEALTHY, "g1": HealthState.HEALTHY}
    asg = schedule(onl, offs, st, crafted_table(), SchedulerConfig(), now=900.0)
    assert [p[:3] for p in asg.pairs] == [("g1", "on-B", "off-C")]
    assert asg.unplaced == ("off-D", "off-E")
    asg = schedule(onl, offs, {"g1": HealthState.HEALTHY}, crafted_table(), SchedulerConfig(), 900.0)
    assert [p[0] for p in asg.pairs] == ["g1"]


def test_memory_quota(cuda):
    from paper_2303_13803_b200 import SchedulerConfig, schedule
    onl, _ = fixture()
    offs = [offline("off-C", 0.25, mem=0.40), offline("off-D", 0.50, mem=0.41),
            offline("off-E", 0.90, mem=0.20)]
    asg = schedule(onl, offs, healthy("g0", "g1"), crafted_table(), SchedulerConfig(), now=900.0)
    placed = {p[2] for p in asg.pairs}
    assert "off-D" not in placed and "off-D" in asg.unplaced and "off-C" in placed


def test_zero_share_and_fixed_sm(cuda):
    from paper_2303_13803_b200 import SchedulerConfig, build_table_from_model, schedule
    onl = [flat_online("on-A", "g0", 0.95), flat_online("on-B", "g1", 0.60)]
    table = build_table_from_model(lambda x, y, z: 0.5, (0.0, 1.0), (0.0, 1.0), (0.0, 1.0))
    asg = schedule(onl, [offline("off-C", 0.25)], healthy("g0", "g1"), table,
                   SchedulerConfig(headroom=0.0), now=900.0)
    assert [p[0] for p in asg.pairs] == ["g1"]
    onl, offs = fixture()
    asg = schedule(onl, offs, healthy("g0", "g1"), crafted_table(),
                   SchedulerConfig(policy="muxflow_fixed_sm", fixed_sm=0.40), now=900.0)
    assert asg.pairs and all(p[3] == 0.40 for p in asg.pairs)


def test_random_match_policy_seeded(cuda):
    from paper_2303_13803_b200 import SchedulerConfig, schedule
    onl, offs = fixture()
    cfg = SchedulerConfig(policy="muxflow_random_match")
    runs = [schedule(onl, offs, healthy("g0", "g1"), crafted_table(), cfg, 900.0, rng=random.Random(7))
            for _ in range(2)]
    assert runs[0] == runs[1] and len(runs[0].pairs) == 2 and len(runs[0].unplaced) == 1


def test_broken_table_aborts(cuda):
    from paper_2303_13803_b200 import SchedulerConfig, SchedulingAborted, schedule
    onl, offs = fixture()
    broken = types.SimpleNamespace(online_sm=None, offline_sm=None, sm_pct=None, values=None)
    with pytest.raises(SchedulingAborted):
        schedule(onl, offs, healthy("g0", "g1"), broken, SchedulerConfig(), now=900.0)


def test_golden_rounds_match_reference(cuda, golden):
    """Assignment equality with the reference's schedule() on synthetic clusters."""
    from paper_2303_13803_b200 import SchedulerConfig, default_table, schedule
    from paper_2303_13803_b200.synth import make_cluster, records
    t = default_table()
    for case in golden["rounds"]["cases"]:
        cl = make_cluster(case["n"], case["m"], seed=case["seed"])
        onl, offs, st = records(cl)
        asg = schedule(onl, offs, st, t, SchedulerConfig(), now=900.0)
        assert [list(p) for p in asg.pairs] == case["pairs"], case["seed"]
        assert list(asg.unplaced) == case["unplaced"]
