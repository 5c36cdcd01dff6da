"""B200-native MuxFlow scheduling round (arXiv 2303.13803).

Drop-in for the hot path of the reference `muxsim` package
(/root/reference/pkg/src/muxsim/__init__.py:10-24): the same `schedule`,
`predict`, `predict_point`, `max_weight_matching` entry points and record
types, with the N x M predictor evaluation and the maximum-weight matching
running as hand-written sm_100a CUDA kernels (libmuxflow.so, C ABI in
include/muxflow.h).  There is no CPU fallback: compute entry points raise if
the library or a B200 is unavailable.
"""

from .core import (HealthState, OfflineWorkload, OnlineWorkload, TraceValidationError,
                   WorkloadProfile)
from .matching import (WEIGHT_FLOOR, BipartiteGraph, Matching, match_dense, max_weight_matching,
                       random_maximal_matching)
from .predictor import (MONOTONE_TOL, PredictionTable, TableError, build_table_from_model,
                        load_table, normalized_throughput, predict, predict_pairs, predict_point,
                        save_table, table_from_dict, table_to_dict)
from .scheduler import (POLICIES, Action, Assignment, SchedulerConfig, SchedulingAborted,
                        dynamic_sm, peak_online_profile, quantize_share, reschedule_actions,
                        round_arrays, schedule)
from .tables import default_table

__all__ = [
    "Action", "Assignment", "BipartiteGraph", "HealthState", "MONOTONE_TOL", "Matching",
    "OfflineWorkload", "OnlineWorkload", "POLICIES", "PredictionTable", "SchedulerConfig",
    "SchedulingAborted", "TableError", "TraceValidationError", "WEIGHT_FLOOR", "WorkloadProfile",
    "build_table_from_model", "default_table", "dynamic_sm", "load_table", "match_dense",
    "max_weight_matching", "normalized_throughput", "peak_online_profile", "predict",
    "predict_pairs", "predict_point", "quantize_share", "random_maximal_matching",
    "reschedule_actions", "round_arrays", "save_table", "schedule", "table_from_dict",
    "table_to_dict",
]
