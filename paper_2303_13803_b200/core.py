"""Input records of the scheduling-round boundary.

`schedule()` takes the reference's record types
(/root/reference/pkg/src/muxsim/core.py:30-136, gpu_state.py:15-20).  These
are compatible stand-ins with the fields and lookups the round reads
(sm_activity, mem_fraction, qps_series, profile_by_qps, qps_at,
profile_for_qps).  `schedule()` duck-types its inputs, so the reference's own
records work unchanged too.
"""

import math
from bisect import bisect_right
from dataclasses import dataclass
from enum import Enum
from typing import Tuple


class TraceValidationError(ValueError):
    """A record failed validation (core.py:10-11)."""


def _fraction(rec, name, value):
    if isinstance(value, bool) or not isinstance(value, (int, float)) or not math.isfinite(value):
        raise TraceValidationError(f"{rec}: {name} must be a finite number, got {value!r}")
    if not 0.0 <= value <= 1.0:
        raise TraceValidationError(f"{rec}: {name} must be in [0, 1], got {value}")


class HealthState(Enum):
    """SysMonitor states (gpu_state.py:15-20); only HEALTHY GPUs get placements."""
    INIT = "init"
    HEALTHY = "healthy"
    UNHEALTHY = "unhealthy"
    OVERLIMIT = "overlimit"
    DISABLED = "disabled"


def is_healthy(state) -> bool:
    """True for HEALTHY of this enum or of any enum whose value is 'healthy'
    (the reference's HealthState included)."""
    if state is None:
        return False
    return getattr(state, "value", None) == "healthy"


@dataclass(frozen=True)
class WorkloadProfile:
    sm_activity: float
    gpu_utilization: float
    sm_occupancy: float
    iter_time_separate: float
    mem_fraction: float

    def __post_init__(self):
        for name in ("sm_activity", "gpu_utilization", "sm_occupancy", "mem_fraction"):
            _fraction("profile", name, getattr(self, name))
        it = self.iter_time_separate
        if isinstance(it, bool) or not isinstance(it, (int, float)) or not math.isfinite(it) or it <= 0:
            raise TraceValidationError(f"profile: iter_time_separate must be > 0, got {it!r}")


@dataclass(frozen=True)
class OnlineWorkload:
    id: str
    gpu_id: str
    base_latency: float
    latency_slo: float
    qps_series: Tuple[Tuple[float, float], ...]
    profile_by_qps: Tuple[Tuple[float, WorkloadProfile], ...]

    def __post_init__(self):
        rec = f"online workload '{self.id}'"
        if not self.qps_series:
            raise TraceValidationError(f"{rec}: qps_series is empty")
        if not self.profile_by_qps:
            raise TraceValidationError(f"{rec}: profiles list is empty")
        ts = [t for t, _ in self.qps_series]
        if any(b <= a for a, b in zip(ts, ts[1:])):
            raise TraceValidationError(f"{rec}: qps_series timestamps must be strictly increasing")
        qs = [q for q, _ in self.profile_by_qps]
        if any(b <= a for a, b in zip(qs, qs[1:])):
            raise TraceValidationError(f"{rec}: profile QPS knots must be strictly increasing")
        if min(q for _, q in self.qps_series) < qs[0]:
            raise TraceValidationError(f"{rec}: qps_series reaches below the lowest profile knot")

    def qps_at(self, t: float) -> float:
        """Step series; before the first knot the first value (core.py:96-100)."""
        i = bisect_right([k[0] for k in self.qps_series], t) - 1
        return self.qps_series[max(i, 0)][1]

    def profile_for_qps(self, qps: float) -> WorkloadProfile:
        """Nearest knot at or below qps (core.py:102-108)."""
        i = bisect_right([k[0] for k in self.profile_by_qps], qps) - 1
        if i < 0:
            raise TraceValidationError(
                f"online workload '{self.id}': no profile knot at or below qps {qps}")
        return self.profile_by_qps[i][1]


@dataclass(frozen=True)
class OfflineWorkload:
    id: str
    submit_time: float
    work_separate: float
    profile: WorkloadProfile
