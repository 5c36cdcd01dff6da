"""The reference CLI's hot-path subcommands and wire formats on the GPU round
(SURVEY.md §8 row f2).

* `schedule --snapshot FILE`: the snapshot JSON of
  /root/reference/pkg/src/muxsim/cli.py:136-221 (`_parse_snapshot`,
  `cmd_schedule`): now, scheduler config, gpu_states, online / offline
  records (sm_activity, mem_fraction), an inline table or a table path.
  Output lines `pairs N`, `pair <gpu> <online> <offline> <share>`,
  `unplaced <offline>`.
* `match --weights FILE`: the `[left, right, weight]` edge list of
  cli.py:267-290, solved by the GPU matcher; output `pair <l> <r>` lines and
  `total <w>`.
* `predict`: the table query / export of cli.py:240-264 (the default table or
  `--table FILE`; `--config` needs the simulator's config and is refused).
Exit codes as cli.py:292-310: 0 ok, 2 invalid input, 3 anything else.  The
simulator subcommands (simulate, validate, gen-trace) are out of scope.
"""

import argparse
import json
import random
import sys
from typing import Dict

from .core import HealthState, OfflineWorkload, OnlineWorkload, TraceValidationError, WorkloadProfile
from .matching import BipartiteGraph, max_weight_matching
from .predictor import TableError, load_table, predict_point, save_table, table_from_dict
from .scheduler import SchedulerConfig, SchedulingAborted, schedule
from .tables import default_table


class ConfigError(ValueError):
    """An invalid command-line combination (the reference's config.py:ConfigError)."""


def _snapshot_profile(entry: Dict) -> WorkloadProfile:
    sm = entry["sm_activity"]
    return WorkloadProfile(sm_activity=sm, gpu_utilization=min(1.0, 1.8 * float(sm)), sm_occupancy=0.5,
                           iter_time_separate=0.1, mem_fraction=entry["mem_fraction"])


def parse_snapshot(doc: Dict):
    """(now, SchedulerConfig, gpu_states, online, offline, table) from a
    snapshot document, with the reference's validation and messages."""
    if not isinstance(doc, dict):
        raise TraceValidationError("snapshot: top level must be an object")
    keys = ("now", "scheduler", "gpu_states", "online", "offline", "table", "table_path")
    unknown = [k for k in doc if k not in keys]
    if unknown:
        raise TraceValidationError(f"snapshot: unknown fields {unknown}")
    for k in ("gpu_states", "online", "offline"):
        if k not in doc:
            raise TraceValidationError(f"snapshot: missing field '{k}'")
    now = float(doc.get("now", 0.0))
    try:
        scfg = SchedulerConfig(**{str(k): v for k, v in doc.get("scheduler", {}).items()})
    except TypeError as e:
        raise TraceValidationError(f"snapshot: scheduler section: {e}") from None
    states = {}
    for gid, name in doc["gpu_states"].items():
        try:
            states[str(gid)] = HealthState(str(name).lower())
        except ValueError:
            raise TraceValidationError(f"snapshot: gpu '{gid}' has unknown state {name!r}") from None
    online = []
    for entry in doc["online"]:
        rec = f"snapshot online '{entry.get('id', '?')}'"
        for k in ("id", "gpu_id", "sm_activity", "mem_fraction"):
            if k not in entry:
                raise TraceValidationError(f"{rec}: missing field '{k}'")
        prof = _snapshot_profile(entry)
        online.append(OnlineWorkload(id=str(entry["id"]), gpu_id=str(entry["gpu_id"]), base_latency=0.02,
                                     latency_slo=0.2, qps_series=((0.0, 1.0),), profile_by_qps=((1.0, prof),)))
    offline = []
    for entry in doc["offline"]:
        rec = f"snapshot offline '{entry.get('id', '?')}'"
        for k in ("id", "sm_activity", "mem_fraction"):
            if k not in entry:
                raise TraceValidationError(f"{rec}: missing field '{k}'")
        offline.append(OfflineWorkload(id=str(entry["id"]), submit_time=float(entry.get("submit_s", 0.0)),
                                       work_separate=float(entry.get("work_s", 3600.0)),
                                       profile=_snapshot_profile(entry)))
    if "table" in doc:
        table = table_from_dict(doc["table"])
    elif "table_path" in doc:
        table = load_table(doc["table_path"])
    else:
        table = default_table()
    return now, scfg, states, online, offline, table


def parse_weights(doc) -> BipartiteGraph:
    """The `match --weights` edge list (cli.py:267-285) as a BipartiteGraph."""
    if not isinstance(doc, list):
        raise ValueError("weights: top level must be a list of [left, right, weight]")
    weights = {}
    for entry in doc:
        try:
            left, right, w = entry
        except (TypeError, ValueError):
            raise ValueError(f"weights: bad entry {entry!r}") from None
        weights[(str(left), str(right))] = float(w)
    return BipartiteGraph(left=tuple(sorted({l for l, _r in weights})),
                          right=tuple(sorted({r for _l, r in weights})), weights=weights)


def _load_json(path, what, err):
    with open(path, "r", encoding="utf-8") as f:
        try:
            return json.load(f)
        except json.JSONDecodeError as e:
            raise err(f"{what} '{path}': invalid JSON ({e})") from e


def cmd_schedule(args) -> int:
    now, scfg, states, online, offline, table = parse_snapshot(_load_json(args.snapshot, "snapshot",
                                                                          TraceValidationError))
    rng = random.Random(f"{args.seed}-match")
    assignment = schedule(online, offline, states, table, scfg, now, rng=rng)
    print(f"pairs {len(assignment.pairs)}")
    for gpu_id, online_id, offline_id, sm in assignment.pairs:
        print(f"pair {gpu_id} {online_id} {offline_id} {sm!r}")
    for offline_id in assignment.unplaced:
        print(f"unplaced {offline_id}")
    return 0


def cmd_match(args) -> int:
    matching = max_weight_matching(parse_weights(_load_json(args.weights, "weights", ValueError)))
    for left, right in matching.pairs:
        print(f"pair {left} {right}")
    print(f"total {matching.total_weight!r}")
    return 0


def cmd_predict(args) -> int:
    if args.config:
        raise ConfigError("predict: --config needs the simulator's configuration (out of scope); use --table")
    table = load_table(args.table) if args.table else default_table()
    coords = (args.online_sm, args.offline_sm, args.sm_pct)
    given = [c for c in coords if c is not None]
    if given and len(given) != 3:
        raise ConfigError("predict: --online-sm, --offline-sm and --sm-pct must be given together")
    if args.save_table:
        save_table(table, args.save_table)
        print(f"wrote {args.save_table}")
    if len(given) == 3:
        print(f"{predict_point(table, args.online_sm, args.offline_sm, args.sm_pct)!r}")
    elif not args.save_table:
        raise ConfigError("predict: nothing to do (give coordinates or --save-table)")
    return 0


def _build_parser():
    p = argparse.ArgumentParser(prog="muxsim", description="MuxFlow scheduling round on the B200")
    sub = p.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("schedule", help="one scheduling round over a snapshot")
    s.add_argument("--snapshot", required=True)
    s.add_argument("--seed", type=int, default=0)
    s.set_defaults(func=cmd_schedule)
    m = sub.add_parser("match", help="maximum-weight matching of an edge list")
    m.add_argument("--weights", required=True)
    m.set_defaults(func=cmd_match)
    q = sub.add_parser("predict", help="query or export the prediction table")
    q.add_argument("--config")
    q.add_argument("--table")
    q.add_argument("--online-sm", type=float)
    q.add_argument("--offline-sm", type=float)
    q.add_argument("--sm-pct", type=float)
    q.add_argument("--save-table")
    q.set_defaults(func=cmd_predict)
    return p


def main(argv=None) -> int:
    args = _build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (TraceValidationError, ConfigError, TableError, FileNotFoundError, IsADirectoryError,
            NotADirectoryError, PermissionError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except (ValueError, SchedulingAborted) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 - CLI boundary
        print(f"error: {e}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
