"""Config-5 replay (BASELINE.json config 5): 100 rounds of the reference's
gen_trace cluster (10k onlines, offline jobs 0 -> 40k), each a full GPU round,
cold (multilevel warm start inside each round) and warm (the previous round's
optimal prices carried across rounds).  Prints one JSON line per mode and
checks the sampled rounds' totals against the CPU goldens.

    python tools/replay.py [rounds] [--check]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2303_13803_b200 import replay  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 100
modes = [m for m in ("cold", "warm") if "--" + m in sys.argv] or ["cold", "warm"]


def progress(rec, _W, _col):
    st = rec["stats"]
    print(f"round {rec['round']}: n {rec['n']} m {rec['m']} warm {rec['warm']} {rec['ms']:.1f} ms "
          f"pops {st['dense_steps']} par {st['par_steps']} levels {st['levels']} total {rec['total_q']}",
          file=sys.stderr, flush=True)

if "--check" in sys.argv:
    os.environ["MUX_SSP_CHECK"] = "1"
gold_path = os.path.join(os.path.dirname(replay.FIXTURE), "replay_cfg5_totals.json")
gold = json.load(open(gold_path))["rounds"] if os.path.exists(gold_path) else {}
res = {}
for warm in [m == "warm" for m in modes]:
    recs = replay.run(rounds=rounds, warm=warm, on_round=progress)
    ms = [r["ms"] for r in recs]
    checked = {str(r["round"]): r["total_q"] == gold[str(r["round"])]["total_q"] for r in recs if str(r["round"]) in gold}
    res[warm] = recs
    print(json.dumps({"mode": "warm" if warm else "cold", "rounds": len(recs), "total_ms": sum(ms),
                      "mean_ms": sum(ms) / len(ms), "max_ms": max(ms),
                      "last_round": {k: recs[-1][k] for k in ("n", "m", "ms", "warm")},
                      "golden_totals_match": checked,
                      "per_round_ms": [round(x, 2) for x in ms],
                      "per_round_m": [r["m"] for r in recs],
                      "dense_pops": [r["stats"]["dense_steps"] for r in recs]}), flush=True)
if len(res) == 2:
    same = all(a["total_q"] == b["total_q"] for a, b in zip(res[False], res[True]))
    print(json.dumps({"warm_equals_cold_totals": same}))
