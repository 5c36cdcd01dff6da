"""The default prediction table (the benchmark fixture).

Tabulates the simulator's ground-truth interference model over the default
9 x 9 x 10 grid, as `default_table(SimConfig())` does
(/root/reference/pkg/src/muxsim/simengine.py:125-203):
rate(d, s, dem) = min(1, occ/dem) * clock(load), occ = min(s, dem),
load = min(1, d + occ), clock = 1 below the 0.5 knee, else
max(0.6, 1 - 0.18 * (load - 0.5) / 0.5).  810 host evaluations, once per run.
"""

from .predictor import PredictionTable, build_table_from_model


def grid(a: float, b: float, n: int):
    """Evenly spaced knots, same float expression as simengine._linspace."""
    if n == 1:
        return (a,)
    return tuple(a + (b - a) * i / (n - 1) for i in range(n))


DEFAULT_ONLINE_SM = grid(0.0, 1.0, 9)
DEFAULT_OFFLINE_SM = grid(0.5, 1.0, 9)
DEFAULT_SM_PCT = grid(0.0, 1.0, 10)


def _clock(load, knee=0.5, slope=0.18, floor=0.6):
    if load <= knee:
        return 1.0
    return max(floor, 1.0 - slope * (load - knee) / (1.0 - knee))


def offline_rate(online_sm: float, offline_sm: float, sm_pct: float) -> float:
    """Unthrottled normalized offline throughput (simengine.py:161-194)."""
    d = min(1.0, max(0.0, online_sm))
    s = min(1.0, max(0.0, sm_pct))
    dem = min(1.0, max(0.0, offline_sm))
    occ = min((1.0 - 0.0) * s, dem)
    load = min(1.0, d + occ)
    c = _clock(load)
    return 0.0 if dem <= 0.0 else min(1.0, occ / dem) * c


def default_table() -> PredictionTable:
    return build_table_from_model(offline_rate, DEFAULT_ONLINE_SM, DEFAULT_OFFLINE_SM,
                                  DEFAULT_SM_PCT, gpu_type="default")
