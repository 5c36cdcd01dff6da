"""Host-side logic of the drop-in boundary (no GPU): config validation, share
sizing, admission, Assignment plumbing, table validation and wire format.
Mirrors the reference's own tests (pkg/tests/test_scheduler.py,
test_predictor.py) for the pieces that stay on the host."""

import random

import numpy as np
import pytest

from paper_2303_13803_b200 import (Action, Assignment, HealthState, OfflineWorkload,
                                   OnlineWorkload, PredictionTable, SchedulerConfig,
                                   SchedulingAborted, TableError, WorkloadProfile, dynamic_sm,
                                   load_table, peak_online_profile, quantize_share,
                                   reschedule_actions, save_table, schedule, table_from_dict,
                                   table_to_dict)
from paper_2303_13803_b200.core import is_healthy
from paper_2303_13803_b200.scheduler import _admissible
from paper_2303_13803_b200.synth import make_cluster, records, shares_for
from paper_2303_13803_b200.tables import default_table


def prof(sm, mem=0.30):
    return WorkloadProfile(sm_activity=sm, gpu_utilization=min(1.0, 1.8 * sm), sm_occupancy=0.5,
                           iter_time_separate=0.1, mem_fraction=mem)


def flat_online(oid, gpu, sm, mem=0.30):
    return OnlineWorkload(id=oid, gpu_id=gpu, base_latency=0.02, latency_slo=0.2,
                          qps_series=((0.0, 100.0),), profile_by_qps=((100.0, prof(sm, mem)),))


def test_dynamic_sm_exact_at_zero_headroom():
    cfg = SchedulerConfig(headroom=0.0)
    assert dynamic_sm(flat_online("u", "g0", 0.20), 900.0, cfg) == 0.80
    assert dynamic_sm(flat_online("u", "g0", 0.80), 900.0, cfg) == 0.20


def test_dynamic_sm_matches_reference_golden(golden):
    cfg = SchedulerConfig()
    for sm, want in golden["dynamic_sm"]["cases"]:
        assert dynamic_sm(flat_online("u", "g", sm), 900.0, cfg) == want
    xs = np.array([c[0] for c in golden["dynamic_sm"]["cases"]])
    assert shares_for(xs).tolist() == [c[1] for c in golden["dynamic_sm"]["cases"]]


def test_quantize_share():
    assert quantize_share(0.80, 0.05) == 0.80
    assert quantize_share(1.0 - 0.80, 0.05) == 0.20
    assert quantize_share(0.0499, 0.05) == 0.0
    assert quantize_share(0.75 - 1e-9, 0.05) == pytest.approx(0.75)


def test_peak_online_profile_window_and_ties():
    profiles = ((100.0, prof(0.20, mem=0.30)), (150.0, prof(0.30, mem=0.33)),
                (200.0, prof(0.50, mem=0.31)), (300.0, prof(0.50, mem=0.32)))
    series = ((0.0, 100.0), (600.0, 200.0), (1200.0, 300.0), (1800.0, 150.0))
    w = OnlineWorkload(id="u", gpu_id="g0", base_latency=0.02, latency_slo=0.2,
                       qps_series=series, profile_by_qps=profiles)
    assert peak_online_profile(w, 0.0, 1900.0).mem_fraction == 0.31
    assert peak_online_profile(w, 1250.0, 1900.0).mem_fraction == 0.32
    assert peak_online_profile(w, 1850.0, 2400.0).sm_activity == 0.30
    assert peak_online_profile(w, -900.0, 0.0).sm_activity == 0.20
    with pytest.raises(ValueError):
        peak_online_profile(w, -900.0, -1.0)


def test_config_validation():
    for kw in (dict(interval=0.0), dict(min_sm=0.6, max_sm=0.5), dict(min_sm=0.0),
               dict(headroom=1.0), dict(quantum=0.0), dict(policy="round_robin"),
               dict(fixed_sm=0.0), dict(mem_quota=1.5)):
        with pytest.raises(ValueError):
            SchedulerConfig(**kw)


def test_admission_boundary_granted():
    offs = [OfflineWorkload("a", 0.0, 1.0, prof(0.3, mem=0.40)),
            OfflineWorkload("b", 0.0, 1.0, prof(0.3, mem=0.41))]
    assert [v.id for v in _admissible(offs, 0.40)] == ["a"]


def test_health_duck_typing():
    assert is_healthy(HealthState.HEALTHY)
    assert not is_healthy(HealthState.UNHEALTHY)
    assert not is_healthy(None)


def test_policies_without_predictor():
    onl = [flat_online("on-B", "g1", 0.60), flat_online("on-A", "g0", 0.20)]
    offs = [OfflineWorkload("off-C", 10.0, 1.0, prof(0.3)), OfflineWorkload("off-A", 5.0, 1.0, prof(0.3)),
            OfflineWorkload("off-B", 5.0, 1.0, prof(0.3))]
    st = {"g0": HealthState.HEALTHY, "g1": HealthState.HEALTHY}
    for policy in ("time_sharing", "pb_time_sharing"):
        asg = schedule(onl, offs, st, None, SchedulerConfig(policy=policy), now=0.0)
        assert asg.pairs == (("g0", "on-A", "off-A", 1.0), ("g1", "on-B", "off-B", 1.0))
        assert asg.unplaced == ("off-C",)
    asg = schedule(onl, offs, st, None, SchedulerConfig(policy="online_only"), now=0.0)
    assert asg.pairs == () and asg.unplaced == ("off-A", "off-B", "off-C")
    with pytest.raises(SchedulingAborted):
        schedule(onl, offs, st, None, SchedulerConfig(), now=0.0)


def test_round_without_pairs_needs_no_gpu():
    # no eligible rows -> no predictor call (scheduler.py:172-180), like the reference
    onl = [flat_online("on-A", "g0", 0.20)]
    offs = [OfflineWorkload("off-C", 0.0, 1.0, prof(0.3))]
    asg = schedule(onl, offs, {"g0": HealthState.UNHEALTHY}, default_table(), SchedulerConfig(), 900.0)
    assert asg.pairs == () and asg.unplaced == ("off-C",)


def test_assignment_and_actions():
    ok = Assignment(pairs=(("g0", "u", "v", 1.0),), unplaced=("w",))
    assert ok.by_offline() == {"v": ("g0", 1.0)}
    for pairs, unplaced in (((("g0", "u", "v", 0.5), ("g0", "x", "y", 0.5)), ()),
                            ((("g0", "u", "v", 0.5), ("g1", "x", "v", 0.5)), ()),
                            ((("g0", "u", "v", 0.0),), ()), ((("g0", "u", "v", 0.5),), ("v",))):
        with pytest.raises(ValueError):
            Assignment(pairs=pairs, unplaced=unplaced)
    prev = Assignment(pairs=(("g0", "u", "A", 0.5), ("g1", "v", "B", 0.4)), unplaced=("C",))
    new = Assignment(pairs=(("g0", "u", "A", 0.3), ("g2", "w", "C", 0.4)), unplaced=("B",))
    assert reschedule_actions(prev, new) == (Action("keep", "A", "g0"), Action("stop", "B", None, "g1"),
                                             Action("start", "C", "g2"))


def test_table_validation_and_wire_format(tmp_path):
    with pytest.raises(TableError):
        PredictionTable("g", (0.5, 0.5), (0.5,), (0.0,), np.zeros((2, 1, 1)))
    with pytest.raises(TableError):
        PredictionTable("g", (0.0,), (0.5,), (0.0,), np.full((1, 1, 1), 1.5))
    with pytest.raises(TableError):
        PredictionTable("g", (0.0,), (0.5,), (0.0, 0.5, 1.0), np.array([[[0.5, 0.4, 0.6]]]))
    t = default_table()
    p1, p2 = tmp_path / "a.json", tmp_path / "b.json"
    save_table(t, str(p1))
    again = load_table(str(p1))
    assert np.array_equal(again.values, t.values) and again.axes == t.axes
    save_table(again, str(p2))
    assert p1.read_bytes() == p2.read_bytes()
    doc = table_to_dict(t)
    doc["vendor"] = "x"
    with pytest.raises(TableError):
        table_from_dict(doc)


def test_default_table_matches_reference(golden):
    t = default_table()
    g = golden["predict_default"]
    assert [list(a) for a in t.axes] == g["axes"]
    assert t.values.reshape(-1).tolist() == g["values"]


def test_synth_records_roundtrip():
    cl = make_cluster(30, 20, seed=3)
    onl, offs, st = records(cl)
    cfg = SchedulerConfig()
    assert [dynamic_sm(u, 900.0, cfg) for u in onl] == cl.share.tolist()
    assert [v.profile.sm_activity for v in offs] == cl.y.tolist()
    assert all(is_healthy(st[u.gpu_id]) for u in onl)
