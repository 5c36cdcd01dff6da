"""Parity at the benchmarked sizes (BASELINE.json configs 2-5) against goldens
computed on the CPU by tests/golden/make_large_golden.py:

  * large_q30_*: scipy.optimize.linear_sum_assignment on the same 30-bit
    integer weights (exact in float64) -> the optimal total.  The GPU round
    (mux_round_dev, with MUX_SSP_CHECK=1: the dense dual certificate
    pi_i + p_j >= a_ij at every level) must reach the same total, and its
    float64 weight matrix must hash to the golden's (bit-identical scoring of
    all N x M pairs).
  * large_f64_4000x4000: the reference algorithm itself (the oracle's C
    restatement of matching.py:45-101 on float64 costs) -> the reference's
    assignment, certified unique (SCC test on the tight-edge digraph).
    Its uniqueness margin is ~1e-12: the reference algorithm itself on 35- /
    40-bit integer weights (large_q35 / large_q40) lands on tied optima 156 /
    8 rows away from it.  The GPU rounds (35 bits = schedule()'s choice at 4k,
    30 bits, 24 bits ~ float32 weights) must reach the integer optimum and
    stay within config 3's tolerance |sum W_ref[gpu] - sum W_ref[ref]| <= N 2^-20.
"""

import glob
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def _load(path):
    with open(path) as f:
        return json.load(f)


def _gold_files(mode):
    return sorted(glob.glob(os.path.join(GOLD, f"large_{mode}_*.json")))


def _round(torch, n, m, seed, qbits, wq=True):
    """One round on device-resident features through mux_round_dev."""
    from paper_2303_13803_b200 import _native as nat, default_table
    from paper_2303_13803_b200.synth import make_cluster
    t = default_table()
    tb, keep = nat.table_struct(t.axes, t.values)
    cl = make_cluster(n, m, seed=seed)
    dev = torch.device("cuda", 0)
    xd, sd, yd = (torch.as_tensor(a, device=dev) for a in (cl.x, cl.share, cl.y))
    dt = torch.int32 if qbits <= 30 else torch.int64
    vec = 4 if qbits <= 30 else 2
    ldw = (m + vec - 1) // vec * vec
    W = torch.empty((n, ldw), dtype=dt, device=dev)
    col = torch.empty(n, dtype=torch.int32, device=dev)
    tot, st = nat.ctypes.c_int64(0), nat.MuxStats()
    nat.check(nat.load().mux_round_dev(nat.context(0), tb, xd.data_ptr(), sd.data_ptr(), n, yd.data_ptr(), m, qbits,
                                       W.data_ptr(), ldw, col.data_ptr(), None, None, 0, nat.ctypes.byref(tot), nat.ctypes.byref(st),
                                       nat.stream_ptr()))
    torch.cuda.synchronize()
    del keep
    return cl, W[:, :m], col.cpu().numpy(), int(tot.value), st.as_dict()


def _scores_f64(torch, cl, rows=None):
    """Exact float64 scores of every pair (optionally a row stripe), on the GPU."""
    from paper_2303_13803_b200 import _native as nat, default_table
    t = default_table()
    tb, keep = nat.table_struct(t.axes, t.values)
    r0, r1 = rows if rows else (0, cl.n)
    dev = torch.device("cuda", 0)
    xd, sd, yd = (torch.as_tensor(a, device=dev) for a in (cl.x[r0:r1], cl.share[r0:r1], cl.y))
    ldw = (cl.m + 1) // 2 * 2
    out = torch.empty((r1 - r0, ldw), dtype=torch.float64, device=dev)
    nat.check(nat.load().mux_score_table(nat.context(0), tb, xd.data_ptr(), sd.data_ptr(), r1 - r0, yd.data_ptr(), cl.m,
                                         nat.MUX_SCORE_EXACT, nat.MUX_W_F64, 0, out.data_ptr(), ldw, nat.stream_ptr()))
    torch.cuda.synchronize()
    return out[:, :cl.m]


def _sha_floor(torch, W):
    W = torch.where(W < 1e-6, torch.zeros((), dtype=W.dtype, device=W.device), W)
    h = hashlib.sha256()
    step = max(1, (1 << 27) // max(1, W.shape[1] * 8))
    for r in range(0, W.shape[0], step):
        h.update(W[r:r + step].contiguous().cpu().numpy().tobytes())
    return h.hexdigest()


@pytest.fixture
def certified(monkeypatch):
    monkeypatch.setenv("MUX_SSP_CHECK", "1")


@pytest.mark.parametrize("path", _gold_files("q30"), ids=lambda p: os.path.basename(p)[6:-5])
def test_round_total_matches_cpu_golden(cuda, certified, path):
    """Configs 2-5 at full size: the optimal total equals scipy LSA's on the CPU."""
    g = _load(path)
    cl, W, col, total, st = _round(cuda, g["n"], g["m"], g["seed"], g["qbits"])
    assert total == g["total_q"], f"GPU total {total} != CPU golden {g['total_q']}"
    # the returned assignment is a matching with exactly that total
    used = col[col >= 0]
    assert len(np.unique(used)) == len(used)
    rows = np.nonzero(col >= 0)[0]
    assert int(W[cuda.as_tensor(rows, device="cuda"), cuda.as_tensor(col[rows].astype(np.int64), device="cuda")]
               .long().sum().item()) == total
    # every pair scored bit-identically to the CPU restatement of predict_point
    assert _sha_floor(cuda, _scores_f64(cuda, cl)) == g["w_sha256"]


def _ref_col(path):
    g = _load(path)
    assert g["unique_optimum"], "golden optimum must be certified unique"
    return g, np.asarray(g["col_of_row"], dtype=np.int64)


F64_4K = os.path.join(GOLD, "large_f64_4000x4000_s0.json")


def _f64_total(W, col):
    return float(sum(W[i, j] for i, j in enumerate(col) if j >= 0))


@pytest.mark.parametrize("q", [35, 40])
def test_int64_round_total_matches_reference_algorithm(cuda, certified, q):
    """Int64 weights at 4k (40 bits = schedule()'s exact-parity quantisation,
    round_qbits; the multilevel solver compiled for int64, csrc/ssp_w64.cu):
    the optimal integer total equals the reference algorithm's on the same
    integers (the oracle's int64 Hungarian, large_q35 / large_q40 goldens)."""
    from paper_2303_13803_b200.matching import round_qbits
    g = _load(os.path.join(GOLD, f"large_q{q}_4000x4000_s0.json"))
    assert round_qbits(max(g["n"], g["m"])) == 40
    _cl, W, col, total, st = _round(cuda, g["n"], g["m"], g["seed"], g["qbits"])
    assert total == g["total_q"]
    assert st["levels"] > 1          # the multilevel solver, not the auction


def test_unique_float64_optimum_needs_more_than_40_bits(cuda):
    """Config 3's unique-optimum check, measured.  The float64 reference
    optimum of the 4k snapshot is certified unique, but only by ~1e-12
    margins: the reference algorithm itself on 35- and 40-bit integer
    weights lands on tied optima that differ from its float64 answer in 156
    and 8 rows (goldens).  The GPU round at schedule()'s 40 bits is one of the
    40-bit optima (same integer total, previous test) and stays within the
    tolerance; the rows it differs in are reported, not asserted."""
    from paper_2303_13803_b200.matching import round_qbits
    g, ref = _ref_col(F64_4K)
    q35 = _load(os.path.join(GOLD, "large_q35_4000x4000_s0.json"))
    q40 = _load(os.path.join(GOLD, "large_q40_4000x4000_s0.json"))
    assert not q35["unique_optimum"] and not q40["unique_optimum"]
    d35 = int(np.sum(np.asarray(q35["col_of_row"]) != ref))
    d40 = int(np.sum(np.asarray(q40["col_of_row"]) != ref))
    assert d35 > 0 and d40 > 0
    cl, _W, col, _total, _st = _round(cuda, g["n"], g["m"], g["seed"], round_qbits(g["n"]))
    Wf = _scores_f64(cuda, cl).cpu().numpy()
    Wf[Wf < 1e-6] = 0.0
    gap = g["total_f64"] - _f64_total(Wf, col)
    assert -1e-9 <= gap <= g["n"] * 2.0 ** -20
    print(f"reference on 35 / 40 bits differs from its float64 optimum in {d35} / {d40} rows; "
          f"GPU 40-bit round: {int(np.sum(col.astype(np.int64) != ref))} rows, float64 gap {gap:.3e}")


def test_schedule_drop_in_at_4k(cuda):
    """The drop-in `schedule()` (records in, Assignment out, scheduler.py:220-241)
    on the 4k x 4k snapshot: a valid Assignment whose float64 total is within
    config 3's tolerance of the reference's (identical placements are pinned
    at <= 128 rows by the golden rounds, tests/test_gpu_scheduler.py)."""
    import time
    from paper_2303_13803_b200 import SchedulerConfig, default_table, schedule
    from paper_2303_13803_b200.synth import make_cluster, records
    g, ref = _ref_col(F64_4K)
    cl = make_cluster(g["n"], g["m"], seed=g["seed"])
    onl, off, states = records(cl)
    table = default_table()
    schedule(onl[:64], off[:64], states, table, SchedulerConfig(), 900.0)   # warm the context
    t0 = time.perf_counter()
    asg = schedule(onl, off, states, table, SchedulerConfig(), 900.0)
    dt = time.perf_counter() - t0
    Wf = _scores_f64(cuda, cl).cpu().numpy()
    Wf[Wf < 1e-6] = 0.0
    row = {u.id: i for i, u in enumerate(onl)}
    col = {v.id: j for j, v in enumerate(off)}
    mine = sum(Wf[row[p[1]], col[p[2]]] for p in asg.pairs)
    assert all(p[3] == float(cl.share[row[p[1]]]) for p in asg.pairs)
    placed = {p[2] for p in asg.pairs}
    assert asg.unplaced == tuple(v.id for v in off if v.id not in placed)
    gap = g["total_f64"] - mine
    assert -1e-9 <= gap <= g["n"] * 2.0 ** -20
    print(f"schedule() 4000 x 4000: {dt * 1e3:.1f} ms, float64 gap to the reference {gap:.3e}")


@pytest.mark.parametrize("qbits", [30, 24])
def test_quantised_rounds_within_config3_tolerance(cuda, qbits):
    """Config 3: a round solved on quantised weights (30 bits; 24 bits = the
    float32 mantissa), evaluated on the reference's float64 weights, is within
    N * 2^-20 of the reference optimum; report how many rows differ."""
    g, ref = _ref_col(F64_4K)
    cl, _W, col, _total, _st = _round(cuda, g["n"], g["m"], g["seed"], qbits)
    Wf = _scores_f64(cuda, cl).cpu().numpy()
    Wf[Wf < 1e-6] = 0.0
    mine = float(sum(Wf[i, j] for i, j in enumerate(col) if j >= 0))
    theirs = float(sum(Wf[i, j] for i, j in enumerate(ref) if j >= 0))
    gap = theirs - mine
    assert abs(theirs - g["total_f64"]) < 1e-9
    assert -1e-9 <= gap <= g["n"] * 2.0 ** -20, f"float64 total gap {gap}"
    print(f"q={qbits}: float64 gap {gap:.3e}, {int(np.sum(col.astype(np.int64) != ref))} rows differ")


@pytest.mark.parametrize("G", [2, 4, 8])
def test_row_sharded_scoring_identical_for_any_gpu_count(cuda, G):
    """Config 3: scoring row stripes independently (as G GPUs would) gives the
    identical weight matrix, hence the identical round, for G in {2, 4, 8}."""
    from paper_2303_13803_b200.synth import make_cluster
    cl = make_cluster(4000, 4000, seed=0)
    full = _scores_f64(cuda, cl)
    bounds = [cl.n * g // G for g in range(G + 1)]
    parts = [_scores_f64(cuda, cl, (bounds[g], bounds[g + 1])) for g in range(G)]
    assert cuda.equal(cuda.cat(parts, 0), full)


def test_round_is_deterministic(cuda):
    """Identical snapshot -> identical assignment (test_matching.py:89-103),
    although the parallel searches race: the canonicalisation fixes the result."""
    a = _round(cuda, 3000, 3000, 7, 30)
    b = _round(cuda, 3000, 3000, 7, 30)
    assert a[3] == b[3]
    assert np.array_equal(a[2], b[2])
