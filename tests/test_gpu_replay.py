"""Config-5 replay rounds (paper_2303_13803_b200.replay) on the GPU: sampled
rounds equal the CPU LSA totals (tests/golden/replay_cfg5_totals.json), and
warm-started rounds (prices carried across rounds) reach the same optimum as
cold ones, with the dense dual certificate on every level (MUX_SSP_CHECK=1)."""

import json
import os

import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "replay_cfg5_totals.json")


def test_replay_rounds_cold_and_warm(cuda, monkeypatch):
    from paper_2303_13803_b200 import replay
    monkeypatch.setenv("MUX_SSP_CHECK", "1")
    k = 15   # rounds 0-11 have fewer jobs than onlines (transposed solve), 12+ more; 13-14 warm
    cold = replay.run(rounds=k, warm=False)
    warm = replay.run(rounds=k, warm=True)
    assert [r["total_q"] for r in cold] == [r["total_q"] for r in warm]
    assert any(r["warm"] for r in warm)
    with open(GOLD) as f:
        gold = json.load(f)["rounds"]
    for r in cold:
        g = gold.get(str(r["round"]))
        if g:
            assert (r["n"], r["m"], r["total_q"]) == (g["n"], g["m"], g["total_q"])
