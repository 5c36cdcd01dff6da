"""GPU parity: the CUDA scoring and matching against the CPU oracle and the
reference's golden vectors.  Everything here calls through libmuxflow.so."""

import random

import numpy as np
import pytest

from oracle import matching_ref, predictor_ref

pytestmark = pytest.mark.gpu


def _table():
    from paper_2303_13803_b200 import default_table
    return default_table()


# ---------------------------------------------------------------- scoring

@pytest.mark.parametrize("n,m,seed", [(1, 1, 0), (7, 5, 1), (64, 64, 2), (333, 1029, 3), (1000, 700, 4)])
def test_exact_scores_bit_identical(cuda, n, m, seed):
    from paper_2303_13803_b200 import predict_pairs
    t = _table()
    rng = np.random.default_rng(seed)
    x, s, y = rng.random(n), rng.random(n), rng.uniform(0.2, 1.0, m)
    # knots, hull edges and exact 0/1
    edge = np.array([0.0, 1.0, 0.5, 0.125, 0.875, 1e-12])
    x[: min(n, 6)] = edge[: min(n, 6)]
    s[: min(n, 6)] = edge[::-1][: min(n, 6)]
    y[: min(m, 4)] = np.array([0.5, 1.0, 0.2, 0.5625])[: min(m, 4)]
    W = predict_pairs(t, x, s, y).cpu().numpy()
    Wo = predictor_ref.predict_pairs_exact(t.axes, t.values, x, s, y)
    assert W.dtype == np.float64
    assert np.array_equal(W, Wo)


def test_golden_predict_points_on_gpu(cuda, golden):
    from paper_2303_13803_b200 import PredictionTable, predict_pairs
    for key in ("predict_default", "predict_linear"):
        g = golden[key]
        axes = tuple(tuple(a) for a in g["axes"])
        t = PredictionTable("g", *axes, np.array(g["values"]).reshape(tuple(len(a) for a in axes)))
        pts = np.array(g["points"])
        W = predict_pairs(t, pts[:, 0], pts[:, 2], pts[:, 1]).cpu().numpy()
        assert np.array_equal(np.diag(W), pts[:, 3])


def test_predict_point_scalar_api(cuda, golden):
    from paper_2303_13803_b200 import predict, predict_point
    from paper_2303_13803_b200.core import WorkloadProfile
    t = _table()
    for x, y, z, want in golden["predict_default"]["points"][:20]:
        assert predict_point(t, x, y, z) == want
    on = WorkloadProfile(0.375, 0.675, 0.5, 0.1, 0.3)
    off = WorkloadProfile(0.75, 1.0, 0.5, 0.1, 0.3)
    assert predict(t, on, off, 0.5) == predict_point(t, 0.375, 0.75, 0.5)


def test_out_of_range_queries_raise(cuda):
    from paper_2303_13803_b200 import TableError, predict_pairs, predict_point
    t = _table()
    for bad in ((1.2, 0.5, 0.5), (0.5, -0.1, 0.5), (0.5, 0.5, float("nan"))):
        with pytest.raises((TableError, ValueError)):
            predict_point(t, *bad)
    with pytest.raises(TableError):
        predict_pairs(t, [0.5, 1.5], [0.5, 0.5], [0.7])


@pytest.mark.parametrize("dtype,qbits", [("int32", 20), ("int32", 30), ("int64", 40)])
def test_quantised_scores(cuda, dtype, qbits):
    from paper_2303_13803_b200 import predict_pairs
    t = _table()
    rng = np.random.default_rng(11)
    x, s, y = rng.random(257), rng.random(257), rng.uniform(0.2, 1.0, 301)
    s[:40] = 0.0          # zero share -> zero weight rows
    Q = predict_pairs(t, x, s, y, dtype=dtype, qbits=qbits).cpu().numpy()
    Wo = predictor_ref.predict_pairs_exact(t.axes, t.values, x, s, y)
    want = np.rint(np.where(Wo >= 1e-6, Wo, 0.0) * 2.0 ** qbits).astype(np.int64)
    assert np.array_equal(Q.astype(np.int64), want)


def test_fast_mode_within_tolerance(cuda):
    from paper_2303_13803_b200 import predict_pairs
    t = _table()
    rng = np.random.default_rng(12)
    x, s, y = rng.random(500), rng.random(500), rng.uniform(0.2, 1.0, 600)
    W = predict_pairs(t, x, s, y, mode="fast", dtype="float32").cpu().numpy().astype(np.float64)
    Wo = predictor_ref.predict_pairs_exact(t.axes, t.values, x, s, y)
    # north_star bar: within 1e-3 relative; fp32 gets ~1e-7
    assert np.max(np.abs(W - Wo) / np.maximum(Wo, 1e-3)) < 1e-5


# ---------------------------------------------------------------- matching

def _graph_from_case(case):
    from paper_2303_13803_b200 import BipartiteGraph
    return BipartiteGraph(tuple(case["left"]), tuple(case["right"]),
                          {(a, b): w for a, b, w in case["edges"]})


def test_golden_matching_totals(cuda, golden):
    from paper_2303_13803_b200 import WEIGHT_FLOOR, max_weight_matching
    for case in golden["matching"]["cases"]:
        g = _graph_from_case(case)
        m = max_weight_matching(g)
        assert m.total_weight == case["total"]
        seen_l, seen_r = set(), set()
        for l, r in m.pairs:
            assert g.weights[(l, r)] >= WEIGHT_FLOOR and l not in seen_l and r not in seen_r
            seen_l.add(l)
            seen_r.add(r)


def test_fig7_example(cuda):
    from paper_2303_13803_b200 import BipartiteGraph, max_weight_matching
    g = BipartiteGraph(("A", "B"), ("C", "D", "E"),
                       {("A", "C"): 0.3, ("A", "D"): 0.8, ("B", "C"): 0.8, ("B", "E"): 0.4})
    m = max_weight_matching(g)
    assert m.pairs == (("A", "D"), ("B", "C")) and m.total_weight == 1.6


def _brute(g):
    from paper_2303_13803_b200 import WEIGHT_FLOOR
    edges = {e: w for e, w in g.weights.items() if w >= WEIGHT_FLOOR}
    lefts = list(g.left)

    def go(i, taken):
        if i == len(lefts):
            return 0.0
        best = go(i + 1, taken)
        for r in g.right:
            if r not in taken and (lefts[i], r) in edges:
                best = max(best, edges[(lefts[i], r)] + go(i + 1, taken | {r}))
        return best
    return go(0, frozenset())


def test_brute_force_1000_instances(cuda):
    """pkg/tests/test_matching.py:45-61 on the GPU solver."""
    from paper_2303_13803_b200 import BipartiteGraph, max_weight_matching
    rng = random.Random(1337)
    for trial in range(1000):
        nl, nr = rng.randint(0, 6), rng.randint(0, 6)
        L = tuple(f"l{i}" for i in range(nl))
        R = tuple(f"r{j}" for j in range(nr))
        w = {(l, r): rng.randrange(65) / 64 for l in L for r in R if rng.random() < 0.7}
        g = BipartiteGraph(L, R, w)
        assert max_weight_matching(g).total_weight == _brute(g), trial


def _pred_Q(n, m, seed, qbits):
    from paper_2303_13803_b200.synth import make_cluster
    t = _table()
    cl = make_cluster(n, m, seed=seed)
    Wo = predictor_ref.predict_pairs_exact(t.axes, t.values, cl.x, cl.share, cl.y)
    return cl, np.rint(np.where(Wo >= 1e-6, Wo, 0.0) * 2.0 ** qbits).astype(np.int64)


def _gpu_match(Q, dtype="int32"):
    import torch
    from paper_2303_13803_b200 import match_dense
    n, m = Q.shape
    vec = 4 if dtype == "int32" else 2
    ldw = max(vec, ((m + vec - 1) // vec) * vec)
    P = np.zeros((n, ldw), dtype=np.int32 if dtype == "int32" else np.int64)
    P[:, :m] = Q
    col, total = match_dense(torch.as_tensor(P, device="cuda"), n, m)
    return col.cpu().numpy(), total


@pytest.mark.parametrize("n,m,seed", [(64, 64, 0), (300, 300, 1), (200, 350, 2), (350, 200, 3),
                                      (1000, 1000, 4)])
def test_predictor_derived_totals(cuda, n, m, seed):
    _, Q = _pred_Q(n, m, seed, 20)
    col, total = _gpu_match(Q)
    want, _ = matching_ref.max_weight_total_int(Q)
    assert total == want
    assert matching_ref.assignment_total_int(Q, col) == want
    used = col[col >= 0]
    assert len(np.unique(used)) == len(used)


def test_uniform_random_weights_unique_optimum_identity(cuda):
    rng = np.random.default_rng(21)
    Q = rng.integers(1, 2 ** 30, size=(500, 500), dtype=np.int64)
    col, total = _gpu_match(Q)
    cost = Q.max() - Q
    ocol, u, v = matching_ref.solve_min_assignment(cost)
    assert matching_ref.is_unique_optimum(cost, ocol, u, v)
    assert total == int(Q[np.arange(500), ocol].sum())
    assert np.array_equal(col, ocol)


def test_int64_weights(cuda):
    _, Q = _pred_Q(120, 90, 5, 24)
    col, total = _gpu_match(Q, dtype="int64")
    want, _ = matching_ref.max_weight_total_int(Q)
    assert total == want


def test_degenerate_inputs(cuda):
    # all-zero weights: nothing emitted; single element; empty side
    col, total = _gpu_match(np.zeros((5, 7), dtype=np.int64))
    assert total == 0 and (col == -1).all()
    col, total = _gpu_match(np.array([[3]], dtype=np.int64))
    assert total == 3 and col.tolist() == [0]
    col, total = _gpu_match(np.full((4, 4), 7, dtype=np.int64))
    assert total == 28 and sorted(col.tolist()) == [0, 1, 2, 3]


def test_deterministic_repeat(cuda):
    _, Q = _pred_Q(400, 400, 6, 20)
    a, ta = _gpu_match(Q)
    b, tb = _gpu_match(Q)
    assert ta == tb and np.array_equal(a, b)


# ---------------------------------------------------------------- full round

@pytest.mark.parametrize("n,m,seed", [(64, 64, 0), (1000, 1000, 1), (500, 800, 2)])
def test_round_total_matches_oracle(cuda, n, m, seed):
    from paper_2303_13803_b200 import round_arrays
    cl, Q = _pred_Q(n, m, seed, 20)
    col, total = round_arrays(_table(), cl.x, cl.share, cl.y, qbits=20)
    want, _ = matching_ref.max_weight_total_int(Q)
    assert total == want
    assert matching_ref.assignment_total_int(Q, col) == want


def test_global_memory_path(cuda, monkeypatch):
    """The auction path used when prices/rows do not fit shared memory."""
    monkeypatch.setenv("MUX_TUNING", "1")
    monkeypatch.setenv("MUX_SOLVER", "auction")
    monkeypatch.setenv("MUX_NO_SMEM", "1")
    for n, m, seed in ((300, 300, 7), (150, 420, 8)):
        _, Q = _pred_Q(n, m, seed, 20)
        col, total = _gpu_match(Q)
        want, _ = matching_ref.max_weight_total_int(Q)
        assert total == want


def test_tail_thresholds(cuda, monkeypatch):
    """Auction: results stay optimal whatever share of the work the single-CTA tail takes."""
    monkeypatch.setenv("MUX_TUNING", "1")
    monkeypatch.setenv("MUX_SOLVER", "auction")
    _, Q = _pred_Q(400, 400, 9, 20)
    want, _ = matching_ref.max_weight_total_int(Q)
    for tail in ("0", "4", "64"):
        monkeypatch.setenv("MUX_TAIL", tail)
        _, total = _gpu_match(Q)
        assert total == want, tail


@pytest.mark.parametrize("kind,n", [("uniform", 2500), ("predictor", 2100)])
def test_large_totals_vs_scipy(cuda, kind, n):
    """Sizes past the 16 x 128-column threshold exercise the threshold top-K
    selection; scipy's exact LSA (cross-checked against the reference on
    dyadic weights) is the oracle here."""
    from scipy.optimize import linear_sum_assignment
    if kind == "uniform":
        Q = np.random.default_rng(1).integers(1, 2 ** 20, size=(n, n), dtype=np.int64)
    else:
        _, Q = _pred_Q(n, n, 5, 20)
    r, c = linear_sum_assignment(Q, maximize=True)
    col, total = _gpu_match(Q)
    assert total == int(Q[r, c].sum())
    assert matching_ref.assignment_total_int(Q, col) == total


def test_scale_invariance_of_pair_choice(cuda):
    """pkg/tests/test_matching.py:116-125: x4 weights -> same pairs, total x4."""
    from paper_2303_13803_b200 import BipartiteGraph, max_weight_matching
    rng = random.Random(5)
    for _ in range(100):
        nl, nr = rng.randint(0, 5), rng.randint(0, 5)
        L = tuple(f"l{i}" for i in range(nl))
        R = tuple(f"r{j}" for j in range(nr))
        w = {(l, r): rng.randrange(65) / 64 for l in L for r in R if rng.random() < 0.7}
        g = BipartiteGraph(L, R, w)
        m1 = max_weight_matching(g)
        m2 = max_weight_matching(BipartiteGraph(L, R, {e: 4.0 * x for e, x in w.items()}))
        assert m1.pairs == m2.pairs
        assert m2.total_weight == 4.0 * m1.total_weight


def test_deterministic_across_input_orderings(cuda):
    """pkg/tests/test_matching.py:89-103."""
    from paper_2303_13803_b200 import BipartiteGraph, max_weight_matching
    rng = random.Random(99)
    for _ in range(200):
        nl, nr = rng.randint(0, 5), rng.randint(0, 5)
        L = [f"l{i}" for i in range(nl)]
        R = [f"r{j}" for j in range(nr)]
        w = {(l, r): rng.randrange(65) / 64 for l in L for r in R if rng.random() < 0.7}
        m1 = max_weight_matching(BipartiteGraph(tuple(L), tuple(R), w))
        rng.shuffle(L)
        rng.shuffle(R)
        items = list(w.items())
        rng.shuffle(items)
        m2 = max_weight_matching(BipartiteGraph(tuple(L), tuple(R), dict(items)))
        assert m1 == m2


def test_golden_pairs_where_optimum_unique(cuda, golden):
    """Identical pair lists wherever the reference's optimum is unique."""
    from paper_2303_13803_b200 import max_weight_matching
    checked = 0
    for case in golden["matching"]["cases"]:
        L, R = sorted(case["left"]), sorted(case["right"])
        if not L or not R:
            continue
        li = {l: i for i, l in enumerate(L)}
        ri = {r: j for j, r in enumerate(R)}
        n = max(len(L), len(R))
        Q = np.zeros((n, n), dtype=np.int64)
        for a, b, x in case["edges"]:
            if x >= 1e-6:
                Q[li[a], ri[b]] = round(x * 64)
        cost = Q.max() - Q
        col, u, v = matching_ref.solve_min_assignment(cost)
        if not matching_ref.is_unique_optimum(cost, col, u, v):
            continue
        m = max_weight_matching(_graph_from_case(case))
        assert [list(p) for p in m.pairs] == case["pairs"]
        checked += 1
    assert checked >= 20


@pytest.mark.parametrize("n,m,seed", [(600, 600, 12), (500, 700, 13), (700, 450, 14)])
def test_async_tail_forced(cuda, monkeypatch, n, m, seed):
    """The concurrent multi-CTA tail (default for n >= 2048) forced on small
    problems: optimal totals, valid assignment."""
    monkeypatch.setenv("MUX_TUNING", "1")
    monkeypatch.setenv("MUX_SOLVER", "auction")
    monkeypatch.setenv("MUX_ASYNC_TAIL", "1")
    _, Q = _pred_Q(n, m, seed, 20)
    col, total = _gpu_match(Q)
    want, _ = matching_ref.max_weight_total_int(Q)
    assert total == want
    assert matching_ref.assignment_total_int(Q, col) == want
    used = col[col >= 0]
    assert len(np.unique(used)) == len(used)


# ------------------------------------------------- tie canonicalisation (a11)

def _dense_graph(W):
    from paper_2303_13803_b200 import BipartiteGraph
    nl, nr = W.shape
    L = tuple(f"l{i:03d}" for i in range(nl))
    R = tuple(f"r{j:03d}" for j in range(nr))
    w = {(L[i], R[j]): float(W[i, j]) for i in range(nl) for j in range(nr) if W[i, j] > 0}
    return BipartiteGraph(L, R, w), L, R


@pytest.mark.parametrize("zeros", [False, True])
def test_canonical_pairs_tie_heavy(cuda, zeros):
    """Dyadic weights from a handful of levels: most instances have many
    optimal matchings; the GPU must emit the reference's canonical one
    (matching.py:173-199), including rectangular (zero-padded) shapes."""
    from paper_2303_13803_b200 import max_weight_matching
    rng = np.random.default_rng(31 + zeros)
    checked = skipped = 0
    for trial in range(250):
        nl, nr = int(rng.integers(1, 24)), int(rng.integers(1, 24))
        levels = int(rng.choice([1, 2, 4, 8]))
        W = rng.integers(1, levels + 1, size=(nl, nr)) / levels
        if zeros:
            W[rng.random((nl, nr)) < 0.35] = 0.0
        want, total, ocol = matching_ref.max_weight_matching_dense(W, return_col=True)
        g, L, R = _dense_graph(W)
        m = max_weight_matching(g)
        assert m.total_weight == total, trial
        if matching_ref.history_sensitive(W, ocol):
            skipped += 1
            continue
        assert list(m.pairs) == [(L[i], R[j]) for i, j in want], trial
        checked += 1
    assert checked >= 150


def test_canonical_golden_pairs_all_cases(cuda, golden):
    """Every golden matching case of the reference (not only the unique
    optima): identical pair lists."""
    from paper_2303_13803_b200 import max_weight_matching
    checked = 0
    for case in golden["matching"]["cases"]:
        L, R = sorted(case["left"]), sorted(case["right"])
        W = np.zeros((len(L), len(R)))
        li = {l: i for i, l in enumerate(L)}
        ri = {r: j for j, r in enumerate(R)}
        for a, b, x in case["edges"]:
            W[li[a], ri[b]] = x
        if L and R:
            _, _, ocol = matching_ref.max_weight_matching_dense(W, return_col=True)
            if matching_ref.history_sensitive(W, ocol):
                continue
        m = max_weight_matching(_graph_from_case(case))
        assert [list(p) for p in m.pairs] == case["pairs"]
        checked += 1
    assert checked >= 100


@pytest.mark.parametrize("n,m,seed", [(400, 400, 41), (300, 520, 42), (520, 300, 43)])
def test_canonical_pairs_predictor_quantised(cuda, n, m, seed):
    """Predictor-derived weights quantised at S = 12 bits (many exact ties):
    the GPU pair list equals the reference restatement's canonical one."""
    from paper_2303_13803_b200 import max_weight_matching
    _, Q = _pred_Q(n, m, seed, 12)
    W = Q / 2.0 ** 12
    want, total, ocol = matching_ref.max_weight_matching_dense(W, return_col=True)
    assert not matching_ref.history_sensitive(W, ocol)
    g, L, R = _dense_graph(W)
    mm = max_weight_matching(g)
    assert mm.total_weight == total
    assert list(mm.pairs) == [(L[i], R[j]) for i, j in want]
