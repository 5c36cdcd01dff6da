"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import matching_ref, predictor_ref


def test_default_table_matches_reference(golden):
    g = golden["predict_default"]
    assert [list(a) for a in predictor_ref.DEFAULT_AXES] == g["axes"]
    vals = predictor_ref.default_table_values()
    assert vals.reshape(-1).tolist() == g["values"]


@pytest.mark.parametrize("key", ["predict_default", "predict_linear"])
def test_predict_point_bit_exact(golden, key):
    g = golden[key]
    axes = tuple(tuple(a) for a in g["axes"])
    vals = np.array(g["values"]).reshape(tuple(len(a) for a in axes))
    for x, y, z, want in g["points"]:
        assert predictor_ref.predict_point(axes, vals, x, y, z) == want


@pytest.mark.parametrize("key", ["predict_default", "predict_linear"])
def test_vectorised_predict_bit_exact(golden, key):
    g = golden[key]
    axes = tuple(tuple(a) for a in g["axes"])
    vals = np.array(g["values"]).reshape(tuple(len(a) for a in axes))
    pts = np.array(g["points"])
    # evaluate the full cross product and read the diagonal pairs back
    W = predictor_ref.predict_pairs_exact(axes, vals, pts[:, 0], pts[:, 2], pts[:, 1])
    assert np.array_equal(np.diag(W), pts[:, 3])


def test_hungarian_restatement_bit_exact(golden):
    for case in golden["hungarian"]["cases"]:
        c = np.array(case["cost"], dtype=np.float64).reshape(len(case["col"]), -1)
        col, u, v = matching_ref.solve_min_assignment(c)
        assert col.tolist() == case["col"]
        assert u.tolist() == case["u"] and v.tolist() == case["v"]
        col2, u2, v2 = matching_ref.solve_min_assignment_py(c)
        assert col2.tolist() == case["col"] and u2.tolist() == case["u"]


def _dense(case):
    L, R = sorted(case["left"]), sorted(case["right"])
    li = {l: i for i, l in enumerate(L)}
    ri = {r: j for j, r in enumerate(R)}
    W = np.zeros((len(L), len(R)))
    for a, b, w in case["edges"]:
        W[li[a], ri[b]] = w
    return L, R, W


def test_matching_restatement_matches_reference(golden):
    for case in golden["matching"]["cases"]:
        L, R, W = _dense(case)
        pairs, total = matching_ref.max_weight_matching_dense(W)
        assert total == case["total"]
        assert [[L[i], R[j]] for i, j in pairs] == case["pairs"]


def test_integer_optimum_matches_reference_totals(golden):
    # the int64 oracle used for GPU parity gives the reference's optimum
    for case in golden["matching"]["cases"]:
        L, R, W = _dense(case)
        if W.size == 0:
            continue
        Q = np.rint(np.where(W >= 1e-6, W, 0) * 64).astype(np.int64)
        total, _ = matching_ref.max_weight_total_int(Q)
        assert total == round(case["total"] * 64)


def test_uniqueness_certificate_small():
    # unique optimum (diagonal dominance) vs an all-ties matrix
    W = np.array([[3, 1], [1, 3]], dtype=np.int64)
    cost = W.max() - W
    col, u, v = matching_ref.solve_min_assignment(cost)
    assert matching_ref.is_unique_optimum(cost, col, u, v)
    W = np.ones((3, 3), dtype=np.int64)
    cost = W.max() - W
    col, u, v = matching_ref.solve_min_assignment(cost)
    assert not matching_ref.is_unique_optimum(cost, col, u, v)
