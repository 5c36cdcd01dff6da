"""GPU parity of the multilevel shortest-path solver (csrc/ssp.cu), the
default matcher for square int32 problems.  Oracles: scipy's exact LSA
(cross-checked against the reference's Hungarian on dyadic weights, SURVEY.md
Appendix A) and the oracle's C restatement of matching.py:45-101.  With
MUX_SSP_CHECK=1 the library also verifies the dense dual certificate
pi_i + p_j >= a_ij (tight on the matching) at every level, which proves
optimality independently of any oracle."""

import functools

import numpy as np
import pytest

from oracle import matching_ref, predictor_ref

pytestmark = pytest.mark.gpu


def _match(Q, keys=None, stats=False):
    import torch
    from paper_2303_13803_b200 import _native as nat
    n, m = Q.shape
    ldw = max(4, (m + 3) // 4 * 4)
    P = np.zeros((n, ldw), dtype=np.int32)
    P[:, :m] = Q
    Wq = torch.as_tensor(P, device="cuda")
    col = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    total = nat.ctypes.c_int64(0)
    st = nat.MuxStats()
    if keys is None:
        rk = ck = None
        rp = cp = None
    else:
        rk = torch.as_tensor(np.asarray(keys[0], dtype=np.float64), device="cuda")
        ck = torch.as_tensor(np.asarray(keys[1], dtype=np.float64), device="cuda")
        rp, cp = rk.data_ptr(), ck.data_ptr()
    nat.check(nat.load().mux_match_keyed(nat.context(0), Wq.data_ptr(), nat.MUX_W_I32, n, m, ldw, rp, cp,
                                         col.data_ptr(), 0, nat.ctypes.byref(total), nat.ctypes.byref(st),
                                         nat.stream_ptr()))
    out = col[:n].cpu().numpy(), int(total.value)
    return out + (st.as_dict(),) if stats else out


def _lsa(Q):
    from scipy.optimize import linear_sum_assignment
    r, c = linear_sum_assignment(Q.astype(np.float64), maximize=True)
    return int(Q[r, c].sum())


def _pred_Q(n, seed, qbits):
    from paper_2303_13803_b200 import default_table
    from paper_2303_13803_b200.synth import make_cluster
    t = default_table()
    cl = make_cluster(n, n, seed=seed)
    W = predictor_ref.predict_pairs_exact(t.axes, t.values, cl.x, cl.share, cl.y)
    return cl, np.rint(np.where(W >= 1e-6, W, 0.0) * 2.0 ** qbits).astype(np.int64)


def _check_assignment(Q, col, total):
    used = col[col >= 0]
    assert len(np.unique(used)) == len(used)
    assert matching_ref.assignment_total_int(Q, col) == total


@pytest.fixture
def certified(monkeypatch):
    monkeypatch.setenv("MUX_SSP_CHECK", "1")


@pytest.fixture
def tuning(monkeypatch):
    """Experiment knobs are honoured only under MUX_TUNING=1."""
    monkeypatch.setenv("MUX_TUNING", "1")


@pytest.mark.parametrize("n,hi,seed", [(2, 5, 0), (7, 100, 1), (33, 3, 2), (50, 1 << 20, 3), (129, 2, 4),
                                       (300, 1000, 5), (777, 50, 6), (1000, 1 << 30, 7)])
def test_random_matrices_vs_lsa(cuda, certified, n, hi, seed):
    """Uniform integer weights, including heavily tied ones (hi = 2, 3)."""
    Q = np.random.default_rng(seed).integers(1, hi, size=(n, n)).astype(np.int64)
    col, total = _match(Q)
    assert total == _lsa(Q)
    _check_assignment(Q, col, total)


@pytest.mark.parametrize("n,q,seed", [(64, 20, 0), (400, 20, 1), (1000, 30, 2), (1500, 24, 3), (2048, 30, 4)])
def test_predictor_rounds_vs_lsa(cuda, certified, n, q, seed):
    """Predictor-derived (near rank-1, degenerate) weights, keyed by the SM demands."""
    cl, Q = _pred_Q(n, seed, q)
    col, total = _match(Q, keys=(cl.x, cl.y))
    assert total == _lsa(Q)
    _check_assignment(Q, col, total)


def test_keys_only_steer_the_warm_start(cuda, certified):
    """Feature keys, row/column-sum keys and adversarial (reversed) keys give the same optimum."""
    cl, Q = _pred_Q(900, 11, 30)
    want = _lsa(Q)
    for keys in ((cl.x, cl.y), None, (-cl.x, cl.y[::-1].copy()), (np.zeros(900), np.zeros(900))):
        col, total = _match(Q, keys=keys)
        assert total == want
        _check_assignment(Q, col, total)


def test_matches_the_oracle_hungarian(cuda, certified):
    """The oracle's C restatement of the reference Kuhn-Munkres on the same integers."""
    for n, q, seed in ((256, 30, 20), (500, 16, 21)):
        _, Q = _pred_Q(n, seed, q)
        want, _ = matching_ref.max_weight_total_int(Q)
        _, total = _match(Q)
        assert total == want


def test_auction_and_ssp_agree(cuda, tuning, monkeypatch):
    """The two GPU solvers (MUX_SOLVER=auction vs the default) reach the same optimum."""
    _, Q = _pred_Q(700, 22, 20)
    _, t_ssp = _match(Q)
    monkeypatch.setenv("MUX_TUNING", "1")
    monkeypatch.setenv("MUX_SOLVER", "auction")
    _, t_auc = _match(Q)
    assert t_ssp == t_auc == _lsa(Q)


@pytest.mark.parametrize("f,base", [("2", "48"), ("4", "48"), ("2", "8"), ("3", "200")])
def test_level_structure_variants(cuda, certified, tuning, monkeypatch, f, base):
    """Coarsening factor and base size change only the work, never the optimum."""
    monkeypatch.setenv("MUX_SSP_F", f)
    monkeypatch.setenv("MUX_SSP_BASE", base)
    cl, Q = _pred_Q(1200, 30, 30)
    _, total = _match(Q, keys=(cl.x, cl.y))
    assert total == _lsa(Q)


@pytest.mark.parametrize("env", [{"MUX_SSP_DORDER": "0"}, {"MUX_SSP_DORDER": "2"}, {"MUX_SSP_SEQ": "0"},
                                 {"MUX_SSP_SEQ": "700"}, {"MUX_SSP_TAILDEF": "0"}, {"MUX_SSP_TAILDEF": "64"},
                                 {"MUX_SSP_FX": "150"}])
def test_scheduling_variants(cuda, certified, tuning, monkeypatch, env):
    """Long-search order, the small-level sequential cut-off, the tail hand-off
    and a fractional level factor change only the work, never the optimum."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cl, Q, want = _pred_case_3000()
    _, total = _match(Q, keys=(cl.x, cl.y))
    assert total == want, env


@functools.lru_cache(maxsize=1)
def _pred_case_3000():
    cl, Q = _pred_Q(3000, 31, 30)
    return cl, Q, _lsa(Q)


def test_long_path_kernels_agree(cuda, certified, tuning, monkeypatch):
    """Cluster (default), single-CTA dense and single-warp sparse long-path modes."""
    cl, Q = _pred_Q(1800, 31, 30)
    want = _lsa(Q)
    for env in ({}, {"MUX_SSP_CLUSTER": "0"}, {"MUX_SSP_CLUSTER": "0", "MUX_SSP_SPARSEX": "1"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        _, total = _match(Q, keys=(cl.x, cl.y))
        assert total == want, env


@pytest.mark.parametrize("env", [{"MUX_SSP_PF": "0"}, {"MUX_SSP_PF": "1"}, {"MUX_SSP_TIES": "0"},
                                 {"MUX_SSP_TIES": "0", "MUX_SSP_PF": "1"}, {"MUX_SSP_L2PF": "1"}] +
                         [{"MUX_SSP_CT": ct} for ct in ("128", "256", "512", "1024")])
def test_long_path_prefetch_variants(cuda, certified, tuning, monkeypatch, env):
    """The long-path kernel (csrc/ssp.cu ssp_rkey_kernel; MUX_SSP_ONE=0 keeps
    every level off the single-SM kernel) with and without tie batching, the
    runner-up row prefetch and the L2 prefetch, and at every CTA size, gives
    the same optimum; the dual certificate is checked at every level
    (MUX_SSP_CHECK=1)."""
    monkeypatch.setenv("MUX_SSP_ONE", "0")
    cl, Q = _pred_Q(2000, 32, 30)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _, total = _match(Q, keys=(cl.x, cl.y))
    assert total == _lsa(Q), env


def test_serial_and_parallel_searches_agree(cuda, certified, tuning, monkeypatch):
    """Lock-based concurrent warp searches vs one search at a time."""
    cl, Q = _pred_Q(1000, 40, 30)
    _, t_par = _match(Q, keys=(cl.x, cl.y))
    monkeypatch.setenv("MUX_SSP_SERIAL", "1")
    _, t_ser = _match(Q, keys=(cl.x, cl.y))
    assert t_par == t_ser == _lsa(Q)


@pytest.mark.slow
def test_certificate_at_4k_many_seeds(cuda, certified):
    """Dense dual certificate at every level, 4k x 4k, several snapshots."""
    from paper_2303_13803_b200 import default_table, round_arrays
    from paper_2303_13803_b200.synth import make_cluster
    t = default_table()
    totals = []
    for seed in range(3):
        cl = make_cluster(4000, 4000, seed=seed)
        col, total, st = round_arrays(t, cl.x, cl.share, cl.y, qbits=30, stats=True)
        assert st["levels"] >= 2
        assert (col >= 0).all()
        totals.append(total)
    assert len(set(totals)) == 3


def test_stats_reported(cuda):
    cl, Q = _pred_Q(1500, 50, 30)
    _, total, st = _match(Q, keys=(cl.x, cl.y), stats=True)
    assert st["total_q"] == total
    assert st["levels"] >= 3
    assert st["par_steps"] > 0
    assert st["ms_parallel"] > 0


# ------------------------------------------------ rectangular rounds (N < M)

@pytest.mark.parametrize("n,m,q,seed", [(1, 5, 20, 0), (50, 64, 20, 1), (300, 900, 20, 2), (999, 1001, 30, 3),
                                        (700, 2800, 30, 4)])
def test_rectangular_predictor_rounds_vs_lsa(cuda, certified, n, m, q, seed):
    """More jobs than online rows: the reference's zero padding rows are implicit
    (rows N..M-1 read a shared zero row); the dual certificate covers them."""
    from paper_2303_13803_b200 import default_table, round_arrays
    from paper_2303_13803_b200.synth import make_cluster
    from scipy.optimize import linear_sum_assignment
    t = default_table()
    cl = make_cluster(n, m, seed=seed)
    W = predictor_ref.predict_pairs_exact(t.axes, t.values, cl.x, cl.share, cl.y)
    Q = np.rint(np.where(W >= 1e-6, W, 0.0) * 2.0 ** q).astype(np.int64)
    r, c = linear_sum_assignment(Q.astype(np.float64), maximize=True)
    col, total, st = round_arrays(t, cl.x, cl.share, cl.y, qbits=q, stats=True)
    assert total == int(Q[r, c].sum())
    _check_assignment(Q, col, total)
    assert st["n_square"] == m


@pytest.mark.parametrize("n,m,hi,seed", [(100, 400, 1000, 0), (333, 500, 3, 1), (64, 1000, 1 << 20, 2)])
def test_rectangular_random_vs_lsa(cuda, certified, n, m, hi, seed):
    Q = np.random.default_rng(seed).integers(0, hi, size=(n, m)).astype(np.int64)
    col, total = _match(Q)
    assert total == _lsa(Q)
    _check_assignment(Q, col, total)


@pytest.mark.parametrize("ties", ["1", "0"])
def test_rectangular_sharded_cluster_tables(cuda, certified, monkeypatch, ties):
    """m above the replicated-table limit (16,384 columns) runs the slice
    kernel (ssp_rkey_slice_kernel: owner and price travel with each warp
    minimum), with and without tie batching; same optimum as the auction."""
    from paper_2303_13803_b200 import default_table, round_arrays
    from paper_2303_13803_b200.synth import make_cluster
    t = default_table()
    cl = make_cluster(1200, 20000, seed=5)
    monkeypatch.setenv("MUX_TUNING", "1")
    monkeypatch.setenv("MUX_SSP_TIES", ties)
    col, total, st = round_arrays(t, cl.x, cl.share, cl.y, qbits=20, stats=True)
    monkeypatch.setenv("MUX_SOLVER", "auction")
    _, t_auc = round_arrays(t, cl.x, cl.share, cl.y, qbits=20)
    assert total == t_auc


@pytest.mark.parametrize("n,m,q,seed", [(5, 1, 20, 0), (64, 50, 20, 1), (900, 300, 20, 2), (1001, 999, 30, 3),
                                        (2800, 700, 30, 4)])
def test_more_rows_than_jobs_vs_lsa(cuda, certified, n, m, q, seed):
    """N > M: the transposed problem (jobs as rows) is solved and the assignment
    and duals are mapped back; the canonicalisation runs in the original orientation."""
    from paper_2303_13803_b200 import default_table, round_arrays
    from paper_2303_13803_b200.synth import make_cluster
    from scipy.optimize import linear_sum_assignment
    t = default_table()
    cl = make_cluster(n, m, seed=seed)
    W = predictor_ref.predict_pairs_exact(t.axes, t.values, cl.x, cl.share, cl.y)
    Q = np.rint(np.where(W >= 1e-6, W, 0.0) * 2.0 ** q).astype(np.int64)
    r, c = linear_sum_assignment(Q.astype(np.float64), maximize=True)
    col, total = round_arrays(t, cl.x, cl.share, cl.y, qbits=q)
    assert total == int(Q[r, c].sum())
    _check_assignment(Q, col, total)


def test_more_rows_than_jobs_random(cuda, certified):
    Q = np.random.default_rng(9).integers(0, 1000, size=(600, 250)).astype(np.int64)
    col, total = _match(Q)
    assert total == _lsa(Q)
    _check_assignment(Q, col, total)


def test_tuning_knobs_are_gated_and_validated(cuda, monkeypatch):
    """Experiment knobs only act under MUX_TUNING=1, and an out-of-range value
    is an error rather than a silent change of the solver."""
    from paper_2303_13803_b200 import _native as nat
    cl, Q = _pred_Q(300, 3, 30)
    want = _lsa(Q)
    monkeypatch.setenv("MUX_SSP_F", "99")        # stray, ungated: ignored
    monkeypatch.setenv("MUX_SOLVER", "bogus")
    assert _match(Q)[1] == want
    monkeypatch.setenv("MUX_TUNING", "1")        # gated: validated
    with pytest.raises(nat.NativeError, match="MUX_SOLVER=bogus"):
        _match(Q)
    monkeypatch.delenv("MUX_SOLVER")
    with pytest.raises(nat.NativeError, match="MUX_SSP_F=99"):
        _match(Q)
    monkeypatch.delenv("MUX_SSP_F")
    monkeypatch.setenv("MUX_SSP_CT", "384")      # in range, not a compiled CTA size
    with pytest.raises(nat.NativeError, match="MUX_SSP_CT must be"):
        _match(Q)


def _match64(Q, keys=None):
    """_match for int64 weights (the solver compiled with 17-bit key indices)."""
    import torch
    from paper_2303_13803_b200 import _native as nat
    n, m = Q.shape
    ldw = max(2, (m + 1) // 2 * 2)
    P = np.zeros((n, ldw), dtype=np.int64)
    P[:, :m] = Q
    Wq = torch.as_tensor(P, device="cuda")
    col = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    total = nat.ctypes.c_int64(0)
    st = nat.MuxStats()
    rp = cp = None
    if keys is not None:
        rk = torch.as_tensor(np.asarray(keys[0], dtype=np.float64), device="cuda")
        ck = torch.as_tensor(np.asarray(keys[1], dtype=np.float64), device="cuda")
        rp, cp = rk.data_ptr(), ck.data_ptr()
    nat.check(nat.load().mux_match_keyed(nat.context(0), Wq.data_ptr(), nat.MUX_W_I64, n, m, ldw, rp, cp,
                                         col.data_ptr(), 0, nat.ctypes.byref(total), nat.ctypes.byref(st),
                                         nat.stream_ptr()))
    return col[:n].cpu().numpy(), int(total.value), st.as_dict()


@pytest.mark.parametrize("n,m,hi,seed", [(300, 300, 1 << 40, 0), (1000, 1000, 1 << 40, 1), (500, 1300, 1 << 38, 2),
                                         (1200, 700, 1 << 40, 3), (800, 800, 5, 4)])
def test_int64_weights_on_the_multilevel_solver(cuda, certified, n, m, hi, seed):
    """Int64 weights (up to 40 bits, square and rectangular both ways, and
    heavily tied) solved by the int64 build of the solver, vs scipy LSA."""
    Q = np.random.default_rng(seed).integers(1, hi, size=(n, m)).astype(np.int64)
    col, total, st = _match64(Q)
    assert total == _lsa(Q)
    assert st["levels"] >= 1                                 # the multilevel solver, not the auction
    _check_assignment(Q, col, total)


def test_int64_predictor_round_vs_oracle_hungarian(cuda, certified):
    """40-bit predictor weights: the integer optimum equals the reference
    algorithm's (the oracle's int64 Hungarian)."""
    cl, Q = _pred_Q(900, 12, 40)
    want, _ = matching_ref.max_weight_total_int(Q)
    col, total, _st = _match64(Q, keys=(cl.x, cl.y))
    assert total == want
    _check_assignment(Q, col, total)
