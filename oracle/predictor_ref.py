"""Oracle restatement of the reference predictor (TEST INFRASTRUCTURE ONLY).

Restates, in plain Python / numpy float64:
  * `_locate`        -- /root/reference/pkg/src/muxsim/predictor.py:74-82
  * `predict_point`  -- predictor.py:85-112 (corner order i, j, k; zero
                        weights skipped; product evaluated left to right as
                        ((wi*wj)*wk)*v; result clamped to [0, 1])
  * the default table of the simulator -- simengine.py:125-203
    (`_linspace`, `ground_truth_step`, `_clock_frac`, `offline_rate_model`,
    `default_table`) and predictor.py:134-153 (`build_table_from_model`).

`predict_pairs_exact` is the vectorised form used to check the GPU scoring
kernel on whole N x M blocks.  Because every term is non-negative, adding a
term whose weight is exactly 0.0 leaves the accumulator bit-identical to the
reference's "skip zero weights" loop, so the vectorised form is bit-exact with
the scalar `predict_point` (pinned by tests/test_oracle_golden.py).
"""

import bisect
import math

import numpy as np


# ---------------------------------------------------------------------------
# scalar restatement (predictor.py:74-112)
# ---------------------------------------------------------------------------

def locate(knots, x):
    """predictor.py:74-82: (lo, hi, frac) with hull clamping."""
    n = len(knots)
    if n == 1 or x <= knots[0]:
        return 0, 0, 0.0
    if x >= knots[-1]:
        return n - 2, n - 1, 1.0
    i = bisect.bisect_right(knots, x) - 1
    return i, i + 1, (x - knots[i]) / (knots[i + 1] - knots[i])


def predict_point(axes, values, online_sm, offline_sm, sm_pct):
    """predictor.py:85-112.  `axes` = (online_sm, offline_sm, sm_pct) tuples."""
    for name, v in (("online_sm", online_sm), ("offline_sm", offline_sm),
                    ("sm_pct", sm_pct)):
        if not 0.0 <= v <= 1.0:
            raise ValueError(f"query {name}={v} outside [0, 1]")
    i0, i1, fi = locate(axes[0], online_sm)
    j0, j1, fj = locate(axes[1], offline_sm)
    k0, k1, fk = locate(axes[2], sm_pct)
    out = 0.0
    for i, wi in ((i0, 1.0 - fi), (i1, fi)):
        if wi == 0.0:
            continue
        for j, wj in ((j0, 1.0 - fj), (j1, fj)):
            if wj == 0.0:
                continue
            for k, wk in ((k0, 1.0 - fk), (k1, fk)):
                if wk == 0.0:
                    continue
                out += wi * wj * wk * float(values[i, j, k])
    return min(1.0, max(0.0, out))


# ---------------------------------------------------------------------------
# vectorised restatement (same arithmetic, whole blocks at once)
# ---------------------------------------------------------------------------

def locate_vec(knots, xs):
    """Vectorised `locate`: arrays (lo, hi, frac) for every query in xs."""
    kn = np.asarray(knots, dtype=np.float64)
    xs = np.asarray(xs, dtype=np.float64)
    n = kn.shape[0]
    lo = np.zeros(xs.shape, dtype=np.int64)
    hi = np.zeros(xs.shape, dtype=np.int64)
    fr = np.zeros(xs.shape, dtype=np.float64)
    if n == 1:
        return lo, hi, fr
    below = xs <= kn[0]
    above = (~below) & (xs >= kn[-1])
    mid = ~(below | above)
    i = np.searchsorted(kn, xs[mid], side="right") - 1
    lo[mid] = i
    hi[mid] = i + 1
    fr[mid] = (xs[mid] - kn[i]) / (kn[i + 1] - kn[i])
    lo[above] = n - 2
    hi[above] = n - 1
    fr[above] = 1.0
    return lo, hi, fr


def predict_pairs_exact(axes, values, x, s, y):
    """W[u, v] = predict_point(x[u], y[v], s[u]) for all pairs, float64, bit-exact."""
    values = np.asarray(values, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    for name, arr in (("online_sm", x), ("offline_sm", y), ("sm_pct", s)):
        if arr.size and not (np.all(arr >= 0.0) and np.all(arr <= 1.0)):
            raise ValueError(f"query {name} outside [0, 1]")
    i0, i1, fi = locate_vec(axes[0], x)
    j0, j1, fj = locate_vec(axes[1], y)
    k0, k1, fk = locate_vec(axes[2], s)
    out = np.zeros((x.shape[0], y.shape[0]), dtype=np.float64)
    for ii, wi in ((i0, 1.0 - fi), (i1, fi)):
        for jj, wj in ((j0, 1.0 - fj), (j1, fj)):
            wij = wi[:, None] * wj[None, :]
            for kk, wk in ((k0, 1.0 - fk), (k1, fk)):
                term = (wij * wk[:, None]) * values[ii[:, None], jj[None, :], kk[:, None]]
                out = out + term
    return np.minimum(1.0, np.maximum(0.0, out))


# ---------------------------------------------------------------------------
# default table (simengine.py:78-86, 125-203; predictor.py:134-153)
# ---------------------------------------------------------------------------

def linspace_ref(a, b, n):
    """simengine.py:125-128."""
    if n == 1:
        return (a,)
    return tuple(a + (b - a) * i / (n - 1) for i in range(n))


DEFAULT_AXES = (linspace_ref(0.0, 1.0, 9), linspace_ref(0.5, 1.0, 9),
                linspace_ref(0.0, 1.0, 10))

# InterferenceParams defaults (simengine.py:78-86) used by the rate model.
LOAD_KNEE = 0.5
CLOCK_SLOPE = 0.18
CLOCK_FLOOR = 0.6


def clock_frac(load, knee=LOAD_KNEE, slope=CLOCK_SLOPE, floor=CLOCK_FLOOR):
    """simengine.py:184-188."""
    if load <= knee:
        return 1.0
    derate = slope * (load - knee) / (1.0 - knee)
    return max(floor, 1.0 - derate)


def offline_rate_model(d, s, dem):
    """simengine.py:161-181 (rate output, throttle 0) / 191-194."""
    d = min(1.0, max(0.0, d))
    s = min(1.0, max(0.0, s))
    thr = 0.0
    dem = min(1.0, max(0.0, dem))
    occ = min((1.0 - thr) * s, dem)
    load = min(1.0, d + occ)
    c = clock_frac(load)
    return 0.0 if dem <= 0.0 else min(1.0, occ / dem) * c


def build_values(model, axes):
    """predictor.py:134-153 (values only; clipped to [0, 1])."""
    ax_i, ax_j, ax_k = axes
    vals = np.empty((len(ax_i), len(ax_j), len(ax_k)), dtype=np.float64)
    for i, xx in enumerate(ax_i):
        for j, yy in enumerate(ax_j):
            for k, zz in enumerate(ax_k):
                vals[i, j, k] = min(1.0, max(0.0, float(model(xx, yy, zz))))
    return vals


def default_table_values():
    """Values of `default_table(SimConfig())` (simengine.py:197-203).

    model(x, y, z) = offline_rate_model(online_sm=x, offline_sm=y, sm_pct=z).
    """
    return build_values(lambda xx, yy, zz: offline_rate_model(xx, zz, yy), DEFAULT_AXES)
