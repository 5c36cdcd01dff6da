"""Oracle restatement of the reference matching (TEST INFRASTRUCTURE ONLY).

Restates /root/reference/pkg/src/muxsim/matching.py on dense arrays:
  * `solve_min_assignment`  -- matching.py:45-101, via oracle/hungarian.c
                               (bit-identical float64 arithmetic) or the
                               pure-numpy `solve_min_assignment_py` for tiny n
  * `repair_path`           -- matching.py:104-145
  * `max_weight_matching_dense` -- matching.py:148-208 (sorted ids are the
                               caller's job: rows/cols here are already in
                               sorted-id order), including the 1e-6 weight
                               floor, zero padding to square, the tie
                               canonicalisation and the "emit only W > 0" rule.
  * `max_weight_total_int`  -- the optimum total of an integer-weight instance
                               (int64 Hungarian), the parity oracle for the
                               GPU auction's quantised totals.
"""

import ctypes
import os

import numpy as np

WEIGHT_FLOOR = 1e-6  # matching.py:19

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            from oracle.build_oracle import build
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        for name, ct in (("hung_solve_f64", ctypes.c_double), ("hung_solve_i64", ctypes.c_int64)):
            fn = getattr(lib, name)
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.POINTER(ct), ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                           ctypes.POINTER(ct), ctypes.POINTER(ct)]
        _lib = lib
    return _lib


def solve_min_assignment(cost):
    """matching.py:45-101 -> (col_of_row int64[n], u, v)."""
    cost = np.ascontiguousarray(cost)
    n = cost.shape[0]
    if cost.dtype == np.int64:
        ct, fn, dt = ctypes.c_int64, "hung_solve_i64", np.int64
    else:
        cost = cost.astype(np.float64, copy=False)
        ct, fn, dt = ctypes.c_double, "hung_solve_f64", np.float64
    col = np.empty(n, dtype=np.int64)
    u = np.empty(n, dtype=dt)
    v = np.empty(n, dtype=dt)
    if n == 0:
        return col, u, v
    rc = getattr(_load(), fn)(cost.ctypes.data_as(ctypes.POINTER(ct)), n,
                              col.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                              u.ctypes.data_as(ctypes.POINTER(ct)),
                              v.ctypes.data_as(ctypes.POINTER(ct)))
    if rc != 0:
        raise MemoryError("oracle hungarian: allocation failed")
    return col, u, v


def solve_min_assignment_py(cost):
    """Literal numpy restatement of matching.py:45-101 (small n only)."""
    n = cost.shape[0]
    INF = float("inf")
    u = np.zeros(n)
    v = np.zeros(n)
    row_of_col = np.full(n, -1, dtype=np.int64)
    minv = np.empty(n)
    way = np.empty(n, dtype=np.int64)
    used = np.empty(n, dtype=bool)
    cand = np.empty(n)
    for i in range(n):
        minv.fill(INF)
        way.fill(-1)
        used.fill(False)
        i0 = i
        j_prev = -1
        while True:
            cur = cost[i0] - u[i0] - v
            better = (~used) & (cur < minv)
            minv[better] = cur[better]
            way[better] = j_prev
            np.copyto(cand, minv)
            cand[used] = INF
            j1 = int(np.argmin(cand))
            delta = cand[j1]
            if used.any():
                u[row_of_col[used]] += delta
                v[used] -= delta
            u[i] += delta
            minv[~used] -= delta
            used[j1] = True
            if row_of_col[j1] < 0:
                break
            i0 = int(row_of_col[j1])
            j_prev = j1
        j = j1
        while True:
            pj = int(way[j])
            if pj < 0:
                row_of_col[j] = i
                break
            row_of_col[j] = row_of_col[pj]
            j = pj
    col_of_row = np.full(n, -1, dtype=np.int64)
    for j in range(n):
        col_of_row[row_of_col[j]] = j
    return col_of_row, u, v


def repair_path(tight, row_of_col, start_row, target_col, banned_row, banned_col, locked_cols):
    """matching.py:104-145."""
    n = tight.shape[0]
    visited_cols = np.zeros(n, dtype=bool)
    visited_cols[banned_col] = True
    visited_cols[locked_cols] = True
    parent_row_of_col = {}
    frontier = [start_row]
    found = False
    while frontier and not found:
        nxt = []
        for r in frontier:
            cols = np.nonzero(tight[r] & ~visited_cols)[0]
            for j in cols:
                visited_cols[j] = True
                parent_row_of_col[int(j)] = r
                if j == target_col:
                    found = True
                    break
                r2 = int(row_of_col[j])
                if r2 != banned_row:
                    nxt.append(r2)
            if found:
                break
        frontier = nxt
    if not found:
        return None
    moves = []
    j = target_col
    while True:
        r = parent_row_of_col[int(j)]
        moves.append((r, int(j)))
        if r == start_row:
            break
        j = int(np.nonzero(row_of_col == r)[0][0])
    return moves


def max_weight_matching_dense(W, canonicalize=True, return_col=False):
    """matching.py:148-208 on a dense (nl x nr) float64 weight array whose
    rows/cols are already in sorted-id order.  Entries < WEIGHT_FLOOR are
    missing edges.  Returns (pairs [(i, j)], total float), plus the full
    square col_of_row when `return_col`."""
    W0 = np.asarray(W, dtype=np.float64)
    nl, nr = W0.shape
    n = max(nl, nr)
    if n == 0:
        return [], 0.0
    Wp = np.zeros((n, n))
    keep = W0 >= WEIGHT_FLOOR
    Wp[:nl, :nr][keep] = W0[keep]
    cost = Wp.max() - Wp
    col_of_row, u, v = solve_min_assignment(cost)
    row_of_col = np.full(n, -1, dtype=np.int64)
    for i in range(n):
        row_of_col[col_of_row[i]] = i
    if canonicalize:
        tight = (cost - u[:, None] - v[None, :]) == 0.0
        locked_cols = np.zeros(n, dtype=bool)
        for i in range(nl):
            j_cur = int(col_of_row[i])
            emitted = j_cur < nr and Wp[i, j_cur] > 0.0
            candidates = np.nonzero(tight[i] & ~locked_cols & (Wp[i] > 0.0))[0]
            for j in candidates:
                j = int(j)
                if emitted and j >= j_cur:
                    break
                moves = repair_path(tight, row_of_col, int(row_of_col[j]), j_cur,
                                    banned_row=i, banned_col=j, locked_cols=locked_cols)
                if moves is None:
                    continue
                for r, jj in moves:
                    row_of_col[jj] = r
                    col_of_row[r] = jj
                row_of_col[j] = i
                col_of_row[i] = j
                j_cur = j
                break
            locked_cols[j_cur] = True
    pairs = []
    total = 0.0
    for i in range(nl):
        j = int(col_of_row[i])
        if j < nr and Wp[i, j] > 0.0:
            pairs.append((i, j))
            total += float(Wp[i, j])
    if return_col:
        return pairs, total, col_of_row
    return pairs, total


def history_sensitive(W, col_of_row):
    """True when a real row ends on a zero-weight REAL column: the one case in
    which the canonical result depends on the reference's own Hungarian
    duals (see csrc/canon.cu), so only totals are comparable."""
    W0 = np.asarray(W, dtype=np.float64)
    nl, nr = W0.shape
    for i in range(nl):
        j = int(col_of_row[i])
        if j < nr and not W0[i, j] >= WEIGHT_FLOOR:
            return True
    return False


def max_weight_total_int(Q):
    """Optimal total of max-weight matching on non-negative int64 weights Q
    (zero = missing edge), with the reference's square zero padding."""
    Q = np.asarray(Q, dtype=np.int64)
    nl, nr = Q.shape
    n = max(nl, nr)
    if n == 0:
        return 0, np.zeros(0, dtype=np.int64)
    P = np.zeros((n, n), dtype=np.int64)
    P[:nl, :nr] = Q
    cost = P.max() - P
    col, _u, _v = solve_min_assignment(cost)
    total = int(P[np.arange(n), col].sum())
    return total, col[:nl]


def assignment_total_int(Q, col_of_row):
    """Total of a (partial) assignment col_of_row (-1 / >= nr = unassigned)."""
    Q = np.asarray(Q, dtype=np.int64)
    nl, nr = Q.shape
    col = np.asarray(col_of_row, dtype=np.int64)
    ok = (col >= 0) & (col < nr)
    return int(Q[np.arange(nl)[ok], col[ok]].sum())


def is_unique_optimum(cost, col_of_row, u, v):
    """Uniqueness certificate (uniq.py recipe): the optimum
    is unique iff the tight-edge digraph (unmatched tight row->col, matched
    col->row) has no cycle, i.e. 2n strongly connected components."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    n = cost.shape[0]
    tight = (cost - u[:, None] - v[None, :]) == 0
    rows, cols = np.nonzero(tight)
    matched = col_of_row[rows] == cols
    # unmatched tight edges row r -> col node n+j; matched edges col n+j -> its row
    row_of_col = np.empty(n, dtype=np.int64)
    row_of_col[col_of_row] = np.arange(n)
    src = np.concatenate([rows[~matched], n + np.arange(n)])
    dst = np.concatenate([n + cols[~matched], row_of_col])
    g = csr_matrix((np.ones(src.shape[0], dtype=np.int8), (src, dst)), shape=(2 * n, 2 * n))
    ncomp, _ = connected_components(g, directed=True, connection="strong")
    return ncomp == 2 * n
