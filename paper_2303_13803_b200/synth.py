"""Synthetic cluster snapshots for benchmarks and parity tests.

One numpy `default_rng(seed)` stream drives every input:
  * online peak SM activity  x_u ~ U(0.15, 0.80)   (gen.py:112-127 range)
  * online memory            ~ U(0.25, 0.62)        (gen.py:30)
  * offline SM demand        y_v ~ U(0.60, 0.98)    (gen.py:34)
  * offline memory           ~ U(0.15, 0.40)        (gen.py:37; all admissible at quota 0.40)
The offered share s_u is the reference `dynamic_sm` formula
(/root/reference/pkg/src/muxsim/scheduler.py:118-135) evaluated in float64,
so the arrays are bit-identical to what the reference computes from the
equivalent `OnlineWorkload` records (`records()` builds those).
"""

from dataclasses import dataclass

import numpy as np

from .scheduler import SchedulerConfig, quantize_share_vec


@dataclass
class Cluster:
    x: np.ndarray          # online peak SM activity, float64 [N]
    share: np.ndarray      # offered SM share, float64 [N] (0 = not eligible)
    online_mem: np.ndarray
    y: np.ndarray          # offline SM demand, float64 [M]
    offline_mem: np.ndarray
    seed: int

    @property
    def n(self):
        return self.x.shape[0]

    @property
    def m(self):
        return self.y.shape[0]


def shares_for(x, cfg=None):
    """dynamic_sm (scheduler.py:123-135) for flat online workloads with peak x."""
    cfg = cfg or SchedulerConfig()
    raw = 1.0 - np.asarray(x, dtype=np.float64) - cfg.headroom
    raw = np.minimum(np.maximum(raw, 0.0), cfg.max_sm)
    share = quantize_share_vec(raw, cfg.quantum)
    share[share < cfg.min_sm] = 0.0
    return share


def make_cluster(n_online, n_offline, seed=0, cfg=None, x_range=(0.15, 0.80)):
    rng = np.random.default_rng(seed)
    x = rng.uniform(x_range[0], x_range[1], n_online)
    online_mem = rng.uniform(0.25, 0.62, n_online)
    y = rng.uniform(0.60, 0.98, n_offline)
    offline_mem = rng.uniform(0.15, 0.40, n_offline)
    return Cluster(x=x, share=shares_for(x, cfg), online_mem=online_mem, y=y,
                   offline_mem=offline_mem, seed=seed)


def records(cl: Cluster, core=None):
    """(online, offline, gpu_states) records equivalent to the arrays.

    `core` is the module providing WorkloadProfile / OnlineWorkload /
    OfflineWorkload / HealthState (this package's `core` by default; the
    golden-vector script passes the reference's modules).
    """
    if core is None:
        from . import core as core_mod
        core = core_mod
    Prof, Onl, Off, HS = core.WorkloadProfile, core.OnlineWorkload, core.OfflineWorkload, core.HealthState
    wn = max(3, len(str(max(cl.n - 1, 0))))
    wm = max(3, len(str(max(cl.m - 1, 0))))
    online, states = [], {}
    for i in range(cl.n):
        sm = float(cl.x[i])
        prof = Prof(sm_activity=sm, gpu_utilization=min(1.0, 1.8 * sm), sm_occupancy=0.5,
                    iter_time_separate=0.1, mem_fraction=float(cl.online_mem[i]))
        gid = f"g{i:0{wn}d}"
        online.append(Onl(id=f"on-{i:0{wn}d}", gpu_id=gid, base_latency=0.02, latency_slo=0.2,
                          qps_series=((0.0, 100.0),), profile_by_qps=((100.0, prof),)))
        states[gid] = HS.HEALTHY
    offline = []
    for j in range(cl.m):
        dem = float(cl.y[j])
        prof = Prof(sm_activity=dem, gpu_utilization=min(1.0, 1.8 * dem), sm_occupancy=0.5,
                    iter_time_separate=0.1, mem_fraction=float(cl.offline_mem[j]))
        offline.append(Off(id=f"off-{j:0{wm}d}", submit_time=0.0, work_separate=3600.0, profile=prof))
    return online, offline, states
