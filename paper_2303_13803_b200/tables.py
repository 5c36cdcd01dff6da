"""The default prediction table (the benchmark fixture).

Tabulates the simulator's ground-truth interference model over the default
9 x 9 x 10 grid, as `default_table(SimConfig())` does
(/root/reference/pkg/src/muxsim/simengine.py:125-203):
rate(d, s, dem) = min(1, occ/dem) * clock(load), occ = min(s, dem),
load = min(1, d + occ), clock = 1 below the 0.5 knee, else
max(0.6, 1 - 0.18 * (load - 0.5) / 0.5).  810 host evaluations, once per run.

Only the table-building part of the reference's simulator config is mirrored
(`InterferenceParams`, `ground_truth_step`, `offline_rate_model`, a
`SimConfig` carrying the grid and the interference parameters); the event
engine itself is out of scope.
"""

from dataclasses import dataclass, field
from typing import Tuple

from .predictor import PredictionTable, build_table_from_model


def grid(a: float, b: float, n: int):
    """Evenly spaced knots, same float expression as simengine._linspace."""
    if n == 1:
        return (a,)
    return tuple(a + (b - a) * i / (n - 1) for i in range(n))


DEFAULT_ONLINE_SM = grid(0.0, 1.0, 9)
DEFAULT_OFFLINE_SM = grid(0.5, 1.0, 9)
DEFAULT_SM_PCT = grid(0.0, 1.0, 10)
DEFAULT_TABLE_ONLINE_SM, DEFAULT_TABLE_OFFLINE_SM, DEFAULT_TABLE_SM_PCT = (DEFAULT_ONLINE_SM, DEFAULT_OFFLINE_SM,
                                                                           DEFAULT_SM_PCT)


@dataclass(frozen=True)
class InterferenceParams:
    """Ground-truth interference shape (simengine.py:75-105); the table uses
    the clock fields, the rest are accepted for constructor compatibility."""

    load_knee: float = 0.5
    clock_slope: float = 0.18
    clock_floor: float = 0.6
    contention_penalty: float = 2.0
    checkpoint_restart_cost: float = 60.0
    control_tick: float = 0.1
    sim_tick: float = 1.0
    online_busy_factor: float = 1.8
    stall_penalty: float = 10.0

    def __post_init__(self):
        if not 0.0 < self.load_knee <= 1.0:
            raise ValueError("load_knee must be in (0, 1]")
        if not 0.0 <= self.clock_slope <= 1.0:
            raise ValueError("clock_slope must be in [0, 1]")
        if not 0.0 < self.clock_floor <= 1.0:
            raise ValueError("clock_floor must be in (0, 1]")
        if self.contention_penalty < 0.0:
            raise ValueError("contention_penalty must be >= 0")
        if self.checkpoint_restart_cost < 0.0:
            raise ValueError("checkpoint_restart_cost must be >= 0")
        if self.control_tick <= 0.0 or self.sim_tick <= 0.0:
            raise ValueError("ticks must be > 0")
        if self.online_busy_factor < 0.0:
            raise ValueError("online_busy_factor must be >= 0")
        if self.stall_penalty < 1.0:
            raise ValueError("stall_penalty must be >= 1")


def _clock(load, p: InterferenceParams = InterferenceParams()):
    if load <= p.load_knee:
        return 1.0
    return max(p.clock_floor, 1.0 - p.clock_slope * (load - p.load_knee) / (1.0 - p.load_knee))


def ground_truth_step(d: float, s: float, throttle_level: float, p: InterferenceParams,
                      offline_sm_demand: float) -> Tuple[float, float, float, float]:
    """One instant of the interference model (simengine.py:161-181):
    (online latency multiplier, offline rate, SM clock fraction, total load)."""
    d = min(1.0, max(0.0, d))
    s = min(1.0, max(0.0, s))
    thr = min(1.0, max(0.0, throttle_level))
    dem = min(1.0, max(0.0, offline_sm_demand))
    occ = min((1.0 - thr) * s, dem)
    overlap = max(0.0, d + occ - 1.0)
    load = min(1.0, d + occ)
    c = _clock(load, p)
    mult = (1.0 / c) * (1.0 + p.contention_penalty * overlap)
    rate = 0.0 if dem <= 0.0 else min(1.0, occ / dem) * c
    return mult, rate, c, load


def offline_rate_model(online_sm: float, offline_sm: float, sm_pct: float,
                       p: InterferenceParams = InterferenceParams()) -> float:
    """Unthrottled normalized offline throughput (simengine.py:191-194)."""
    return ground_truth_step(online_sm, sm_pct, 0.0, p, offline_sm)[1]


def offline_rate(online_sm: float, offline_sm: float, sm_pct: float) -> float:
    return offline_rate_model(online_sm, offline_sm, sm_pct)


@dataclass(frozen=True)
class SimConfig:
    """The table-building fields of the reference's SimConfig (simengine.py:137-158)."""

    interference: InterferenceParams = field(default_factory=InterferenceParams)
    table_online_sm: Tuple[float, ...] = DEFAULT_ONLINE_SM
    table_offline_sm: Tuple[float, ...] = DEFAULT_OFFLINE_SM
    table_sm_pct: Tuple[float, ...] = DEFAULT_SM_PCT


def default_table(cfg: SimConfig = None) -> PredictionTable:
    """Tabulate the ground-truth model over the configured grid (simengine.py:197-203)."""
    cfg = cfg or SimConfig()
    p = cfg.interference
    return build_table_from_model(lambda x, y, z: offline_rate_model(x, y, z, p),
                                  cfg.table_online_sm, cfg.table_offline_sm, cfg.table_sm_pct,
                                  gpu_type="default")
