"""Host-side wire formats of the reference CLI (paper_2303_13803_b200/cli.py,
restating /root/reference/pkg/src/muxsim/cli.py:136-221, 267-290): snapshot
and edge-list parsing and their validation.  No GPU: every malformed input is
rejected before any device work (the subcommands themselves run in
tests/ref_suite/test_ref_cli.py on the B200)."""

import json

import pytest

from paper_2303_13803_b200.cli import main, parse_snapshot, parse_weights
from paper_2303_13803_b200.core import HealthState, TraceValidationError

SNAPSHOT = {
    "now": 900.0,
    "scheduler": {"policy": "muxflow"},
    "gpu_states": {"g0": "healthy", "g1": "HEALTHY"},
    "online": [{"id": "on-A", "gpu_id": "g0", "sm_activity": 0.20, "mem_fraction": 0.30},
               {"id": "on-B", "gpu_id": "g1", "sm_activity": 0.60, "mem_fraction": 0.30}],
    "offline": [{"id": "off-C", "sm_activity": 0.25, "mem_fraction": 0.20, "submit_s": 5.0}],
}


def test_snapshot_fields():
    now, cfg, states, online, offline, table = parse_snapshot(SNAPSHOT)
    assert now == 900.0 and cfg.policy == "muxflow"
    assert states == {"g0": HealthState.HEALTHY, "g1": HealthState.HEALTHY}
    assert [u.id for u in online] == ["on-A", "on-B"] and online[1].profile_for_qps(1.0).sm_activity == 0.60
    assert offline[0].submit_time == 5.0 and offline[0].profile.gpu_utilization == pytest.approx(0.45)
    assert table.values.shape == (9, 9, 10)          # default table when none is given


@pytest.mark.parametrize("bad", [
    dict(SNAPSHOT, gpu_states={"g0": "wobbly"}),
    dict(SNAPSHOT, scheduler={"warp": 9}),
    {k: v for k, v in SNAPSHOT.items() if k != "online"},
    dict(SNAPSHOT, extra=1),
    dict(SNAPSHOT, online=[{"id": "x", "gpu_id": "g0", "sm_activity": 0.2}]),
    [],
])
def test_snapshot_rejects(bad):
    with pytest.raises(TraceValidationError):
        parse_snapshot(bad)


def test_weights_and_exit_codes(tmp_path):
    g = parse_weights([["A", "C", 0.3], ["A", "D", 0.8], ["B", "C", 0.8]])
    assert g.left == ("A", "B") and g.right == ("C", "D") and g.weights[("A", "D")] == 0.8
    for doc in ([["A", "C"]], {"A": 1}):
        p = tmp_path / "w.json"
        p.write_text(json.dumps(doc))
        assert main(["match", "--weights", str(p)]) == 2
    p = tmp_path / "s.json"
    p.write_text(json.dumps(dict(SNAPSHOT, extra=1)))
    assert main(["schedule", "--snapshot", str(p)]) == 2
    assert main(["predict", "--online-sm", "0.5"]) == 2
    assert main(["schedule", "--snapshot", str(tmp_path / "missing.json")]) == 2
