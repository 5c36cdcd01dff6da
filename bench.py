"""Benchmark: one MuxFlow scheduling round (predict + optimal match) at 10k x 10k.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--n 10000] [--m 10000] [--qbits 30]

A step is one full round over one synthetic cluster snapshot:
exact float64 scoring of every (online, offline) pair into int32 weights
rint(w * 2^30) (csrc/score.cu; 30 bits is the finest int32 quantisation and the
closest to the reference's float64 weights -- SURVEY's S = 20 is available
with --qbits 20 and has ~14x more tight (tied) edges), then the exact
maximum-weight matching by the multilevel shortest-path solver (csrc/ssp.cu:
stratified coarse levels, c-transform warm prices, parallel warp Dijkstras and
a single-CTA dense Dijkstra for long paths) and the tie canonicalisation
(csrc/canon.cu).  `value` is ms per round with the
feature arrays already resident in HBM (device-timed with CUDA events on the
launching stream); `e2e` is the same round through the C-ABI `mux_round` with
HOST feature arrays (H2D of features and D2H of col_of_row inside the timed
region).  With N GPUs each rank solves its own snapshot (seed + rank): the
round does not shard usefully, so `value` stays the per-round
latency (max over ranks) and replica throughput is reported separately.
When tests/golden holds the CPU-computed optimal total for the workload
(scipy LSA on the same integer weights), the round's total must equal it.

`--impl reference` runs the unmodified reference package (baseline/_ref,
pip-installed from /root/reference/pkg) on one host core: measured
`schedule()` rounds at 64^2 (the timed steps) and 256^2..1024^2, extrapolated
to the metric's 10k x 10k round (hours of CPU time).
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per scheduling round (predict+match) at 10k×10k; pair scores/sec"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=10000)
    p.add_argument("--m", type=int, default=10000)
    p.add_argument("--qbits", type=int, default=30)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-mlp", action="store_true")
    p.add_argument("--no-schedule", action="store_true")
    return p.parse_args()


def bf16_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)["bf16_tflops"]
    except Exception:
        return 1590.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU reference arm: the unmodified reference `muxsim` package
# ---------------------------------------------------------------------------

def load_reference():
    """Import the reference package unmodified: baseline/_ref (pip-installed
    from /root/reference/pkg, travels to the GPU box) or, in the build
    container only, /root/reference/pkg/src.  Returns (modules, path) or None."""
    import importlib
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if not os.path.isfile(os.path.join(path, "muxsim", "scheduler.py")):
            continue
        sys.path.insert(0, path)
        try:
            mods = {k: importlib.import_module(f"muxsim.{k}")
                    for k in ("core", "gpu_state", "scheduler", "simengine", "matching", "predictor")}
        finally:
            sys.path.remove(path)
        if not os.path.abspath(mods["scheduler"].__file__).startswith(os.path.abspath(path)):
            continue
        return mods, path
    return None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_round_ms(ref, n, m, seed):
    """Wall time of one reference `schedule()` round (scheduler.py:220-241) on the
    synthetic snapshot make_cluster(n, m, seed): records built with the
    reference's own types, default_table(SimConfig()), SchedulerConfig(), now=900."""
    from paper_2303_13803_b200.synth import make_cluster, records

    class Core:
        WorkloadProfile = ref["core"].WorkloadProfile
        OnlineWorkload = ref["core"].OnlineWorkload
        OfflineWorkload = ref["core"].OfflineWorkload
        HealthState = ref["gpu_state"].HealthState

    cl = make_cluster(n, m, seed=seed)
    onl, off, states = records(cl, core=Core)
    table = ref["simengine"].default_table(ref["simengine"].SimConfig())
    cfg = ref["scheduler"].SchedulerConfig()
    t0 = time.perf_counter()
    asg = ref["scheduler"].schedule(onl, off, states, table, cfg, 900.0)
    dt = time.perf_counter() - t0
    return dt * 1e3, asg, (cl, table)


def reference_match_ms(ref, cl, table):
    """Wall time of the reference's public max_weight_matching (matching.py:148-208)
    alone, on the graph its round builds (weights from its public predict_point)."""
    mt, pr = ref["matching"], ref["predictor"]
    L = [f"u{i}" for i in range(cl.n)]
    R = [f"v{j}" for j in range(cl.m)]
    w = {}
    for i in range(cl.n):
        for j in range(cl.m):
            x = pr.predict_point(table, float(cl.x[i]), float(cl.y[j]), float(cl.share[i]))
            if x > 0.0:
                w[(L[i], R[j])] = x
    g = mt.BipartiteGraph(tuple(L), tuple(R), w)
    t0 = time.perf_counter()
    mt.max_weight_matching(g)
    return (time.perf_counter() - t0) * 1e3, w


def lsa_ms(cl, table_vals_fn):
    from scipy.optimize import linear_sum_assignment
    W = table_vals_fn(cl)
    t0 = time.perf_counter()
    linear_sum_assignment(W, maximize=True)
    return (time.perf_counter() - t0) * 1e3


def reference_estimate(ref, n, m, seed, k1, k2):
    """Measured reference rounds at k1^2 and k2^2 (k2 = 2 k1) and the solver
    alone on both; extrapolated to n x m: predict per pair x N*M plus the
    Kuhn-Munkres time x (n/k2)^e, e fitted on the k1 -> k2 solves."""
    rounds, solves = {}, {}
    for k in (k1 // 2, k1, k2):
        ms, _asg, (cl, table) = reference_round_ms(ref, k, k, seed)
        rounds[k] = ms
        if k >= k1:
            solves[k], _w = reference_match_ms(ref, cl, table)
    e = math.log(solves[k2] / solves[k1]) / math.log(k2 / k1)
    e = min(3.2, max(2.5, e))
    pred_per_pair = max(0.0, rounds[k2] - solves[k2]) / float(k2 * k2)
    n_sq = max(n, m)
    est = pred_per_pair * n * m + solves[k2] * (n_sq / float(k2)) ** e
    sample = (f"reference muxsim.scheduler.schedule(), 1 core ({cpu_model()}): measured rounds "
              f"{', '.join(f'{k}^2 {v / 1e3:.2f} s' for k, v in rounds.items())}; solver alone "
              f"{', '.join(f'{k}^2 {v / 1e3:.2f} s' for k, v in solves.items())} (fit n^{e:.2f}); "
              f"predict {pred_per_pair * 1e3:.2f} us/pair; EXTRAPOLATED to {n}x{m}")
    measured = {"round_ms": rounds, "solve_ms": solves, "solve_exponent": e, "predict_us_per_pair": pred_per_pair * 1e3}
    return est, sample, measured


def pin_one_core():
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except (AttributeError, OSError):
        pass
    return 1


def run_reference(args, rank, world):
    """--impl reference: the reference's own scheduler on this host's cores.

    Rank 0 alone runs (other ranks exit at once).  The reference is
    single-threaded Python + numpy; it is pinned to one core.  Each timed
    step is one full `schedule()` round at 64 x 64 (BASELINE config 1),
    measured.  The 10k x 10k metric is out of reach (~hours), so the
    line's value is extrapolated from MEASURED rounds at 256^2 / 512^2 /
    1024^2 split into phases: predict loop (per pair, x N*M) and the
    Kuhn-Munkres solve (x (n/1024)^e, e fitted on the measured 512 -> 1024
    solves).  scipy's linear_sum_assignment (C) is timed beside it."""
    if rank != 0:
        return
    got = load_reference()
    if got is None:
        print(json.dumps({"impl": "reference", "unavailable": "reference muxsim package not found in baseline/_ref"}))
        return
    ref, ref_path = got
    cores = pin_one_core()
    small = []
    for s in range(args.warmup + args.steps):
        ms, _asg, _ = reference_round_ms(ref, 64, 64, args.seed + s)
        if s >= args.warmup:
            small.append(ms)
    est, sample, measured = reference_estimate(ref, args.n, args.m, args.seed, 512, 1024)
    # scipy LSA (single-thread C, not the reference) on the same weights
    from oracle import predictor_ref
    from paper_2303_13803_b200.synth import make_cluster
    vals = predictor_ref.default_table_values()

    def wfn(cl):
        return predictor_ref.predict_pairs_exact(predictor_ref.DEFAULT_AXES, vals, cl.x, cl.share, cl.y)
    measured["scipy_lsa_ms"] = {k: lsa_ms(make_cluster(k, k, seed=args.seed), wfn) for k in (1024, 2048)}
    measured["round_64_ms"] = small
    sample = f"{sample}; package from {os.path.relpath(ref_path, ROOT) if ref_path.startswith(ROOT) else ref_path}"
    v = est
    line = {"metric": METRIC, "value": v, "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args),
            "impl": "reference", "extrapolated": True,
            "cpu_baseline": {"value": v, "unit": "ms", "cores": cores, "kind": "reference", "sample": sample,
                             "cpu_model": cpu_model(), "nproc": os.cpu_count()},
            "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "measured": measured,
            "pair_scores_per_s": args.n * args.m / (v / 1e3)}
    print(json.dumps(line), flush=True)


def ncu_traffic():
    """DRAM bytes per launch of the dominant kernel from the newest committed ncu capture."""
    for rnd, name in (("r03", "ncu_rkey_traffic.json"), ("r02", "ncu_cluster_traffic.json")):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, name)) as f:
                return json.load(f)["dram_bytes_per_launch"], rnd
        except Exception:
            continue
    return None, None


def workload_config(args):
    """Identical in both arms (the driver compares them)."""
    return {"workload": f"{args.n}x{args.m} scheduling round (predict + optimal match)",
            "n_online": args.n, "n_offline": args.m, "seed": args.seed,
            "inputs": "synth.make_cluster(n, m, seed), default table; weight matrix (400 MB) > L2"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2303_13803_b200 import _native as nat
    from paper_2303_13803_b200 import default_table, round_arrays
    from paper_2303_13803_b200.synth import make_cluster

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    lib = nat.load()
    ctx = nat.context(local_rank)
    stream = torch.cuda.current_stream(dev)
    sptr = nat.ctypes.c_void_p(stream.cuda_stream)
    table = default_table()
    tb, keep = nat.table_struct(table.axes, table.values)
    n, m, q = args.n, args.m, args.qbits
    ldw = ((m + 3) // 4) * 4
    # each rank: its own replica snapshot (different seed); inputs resident in HBM
    cl = make_cluster(n, m, seed=args.seed + rank)
    xd = torch.as_tensor(cl.x, device=dev)
    sd = torch.as_tensor(cl.share, device=dev)
    yd = torch.as_tensor(cl.y, device=dev)
    Wq = torch.empty((n, ldw), dtype=torch.int32, device=dev)
    col = torch.empty(n, dtype=torch.int32, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    total = nat.ctypes.c_int64(0)
    st = nat.MuxStats()

    def step():
        # one fused round on the HBM-resident snapshot: exact scoring into Wq,
        # the multilevel solve (ordered by the online / offline SM demands), the
        # tie canonicalisation
        nat.check(lib.mux_round_dev(ctx, tb, xd.data_ptr(), sd.data_ptr(), n, yd.data_ptr(), m, q, Wq.data_ptr(), ldw,
                                    col.data_ptr(), None, None, 0, nat.ctypes.byref(total), nat.ctypes.byref(st), sptr))
        return st.as_dict(), int(total.value)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    times, match_ms, stats_all = [], [], []
    for _ in range(args.steps):
        flush.zero_()                                   # L2 flush between timed iterations
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        s, tot = step()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        match_ms.append(s["ms_match"])
        stats_all.append(s)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    t_step = sum(times) / len(times)
    if world > 1:
        tt = torch.tensor([t_step], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
        dist.barrier()

    # sanity: total of the returned assignment equals the reported optimum
    Qh = Wq[:, :m]
    colh = col.long()
    ok = colh >= 0
    got = int(Qh[torch.arange(n, device=dev)[ok], colh[ok]].long().sum().item())
    assert got == stats_all[-1]["total_q"], "assignment total != reported total"

    # e2e through the C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        for _ in range(1):
            round_arrays(table, cl.x, cl.share, cl.y, qbits=q)
        ts = []
        for _ in range(max(1, min(args.steps, 3))):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            round_arrays(table, cl.x, cl.share, cl.y, qbits=q)
            ts.append((time.perf_counter() - t0) * 1e3)
        e2e_ms = sum(ts) / len(ts)
        if world > 1:
            tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item())
        e2e = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": (2 * n + m) * 8,
               "d2h_bytes_per_step": n * 4, "path": "mux_round C-ABI with host feature arrays (H2D + D2H in the timed region)",
               "per_rank": True}

    # MLP plugin (tcgen05) scoring of the same N x M pairs: tensor-core roofline
    # the drop-in call a reference user makes: schedule(records) -> Assignment,
    # host record handling included (scheduler.py:220-241), at configs 2 and 3
    sched_line = None
    if not args.no_schedule and rank == 0:
        from paper_2303_13803_b200 import SchedulerConfig, schedule
        from paper_2303_13803_b200.matching import round_qbits
        from paper_2303_13803_b200.synth import records
        sched_line = {}
        for k in (1000, 4000):
            c = make_cluster(k, k, seed=args.seed)
            onl, off, states = records(c)
            schedule(onl, off, states, table, SchedulerConfig(), 900.0)
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                asg = schedule(onl, off, states, table, SchedulerConfig(), 900.0)
                ts.append((time.perf_counter() - t0) * 1e3)
            sched_line[f"{k}x{k}"] = {"ms": statistics.median(ts), "pairs": len(asg.pairs),
                                      "qbits": round_qbits(k),
                                      "solver": "multilevel SSP, int64 weights" if round_qbits(k) > 30 else "multilevel SSP, int32 weights"}

    mlp_line = None
    if not args.no_mlp:
        from paper_2303_13803_b200.mlp import MlpPredictor
        mlp = MlpPredictor.random(args.seed)
        rng = np.random.default_rng(args.seed)
        on = torch.as_tensor(np.stack([np.minimum(1.0, 1.8 * cl.x), cl.x, np.full(n, 0.5),
                                       rng.uniform(0.01, 0.04, n)], axis=1), device=dev)
        off = torch.as_tensor(np.stack([np.minimum(1.0, 1.8 * cl.y), cl.y, np.full(m, 0.5),
                                        np.full(m, 0.1)], axis=1), device=dev)
        Wm = torch.empty((n, ldw), dtype=torch.float32, device=dev)
        st_m, keep_m = mlp.struct()

        def mlp_step():
            nat.check(lib.mux_score_mlp(ctx, nat.ctypes.byref(st_m), on.data_ptr(), sd.data_ptr(), n,
                                        off.data_ptr(), m, nat.MUX_W_F32, 0, Wm.data_ptr(), ldw, sptr))
        for _ in range(2):
            mlp_step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            mlp_step()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        mlp_ms = sorted(ts)[len(ts) // 2]
        flops = 2.0 * 64 * 64 * 2 * n * m + 4.0 * 64 * n * m
        issued = 2.0 * (144 + 128) * 64 * n * m      # tensor flops issued: K = 64 hi + 64 lo (+ 16 bias in layer 2)
        mlp_line = {"ms": mlp_ms, "tflops": flops / (mlp_ms / 1e3) / 1e12, "flops": flops,
                    "tensor_tflops_issued": issued / (mlp_ms / 1e3) / 1e12,
                    "note": "algorithmic flops (16.6 kFLOP/pair); layers 2-3 as tcgen05 kind::f16 M128 N64, "
                            "split fp16 activations (hi + lo): K = 144 / 128, layer 3 A operand in TMEM, fp32 TMEM accumulate"}

    if rank != 0:
        return
    hbm, peak_kind = peaks()
    # dominant kernel: ssp_rkey_kernel (csrc/ssp.cu), the thread-block-cluster
    # Dijkstra that runs the long augmenting paths of every level.  Algorithmic
    # bytes = one weight row (4*m_level) per pop (SURVEY §8d's per-row-read
    # unit), summed over its pops; time = its CUDA-event duration on the
    # launching stream inside the solve.  `traffic`: DRAM bytes per launch from
    # the committed ncu --set full capture of the same kernel (profiles/).
    dense_ms = sum(x["ms_dense"] for x in stats_all) / len(stats_all)
    dense_bytes = sum(x["dense_bytes"] for x in stats_all) / len(stats_all)
    achieved = dense_bytes / (dense_ms / 1e3) / 1e9 if dense_ms > 0 else 0.0
    auc_ms = sum(match_ms) / len(match_ms)
    traffic, traffic_src = ncu_traffic()
    cpu = None
    if not args.no_cpu:
        got = load_reference()
        if got is not None:
            # bounded sample (~10 s): measured reference rounds at 128^2..512^2
            with_aff = os.sched_getaffinity(0)
            cores = pin_one_core()
            cpu_ms, sample, measured = reference_estimate(got[0], n, m, args.seed, 256, 512)
            os.sched_setaffinity(0, with_aff)
            cpu = {"value": cpu_ms, "unit": "ms", "cores": cores, "kind": "reference", "sample": sample,
                   "measured": measured, "extrapolated": True}
    s = stats_all[-1]
    value = t_step
    parity = None
    gpath = os.path.join(ROOT, "tests", "golden", f"large_q{q}_{n}x{m}_s{args.seed}.json")
    if rank == 0 and os.path.exists(gpath):
        with open(gpath) as f:
            gold = json.load(f)["total_q"]
        parity = {"total_q": stats_all[-1]["total_q"], "golden_total_q": gold, "golden": os.path.relpath(gpath, ROOT),
                  "match": stats_all[-1]["total_q"] == gold}
        assert parity["match"], f"optimal total {stats_all[-1]['total_q']} != golden {gold}"
    line = {
        "metric": METRIC, "value": value, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32 (f64 scoring)", "data": "synthetic",
        "config": workload_config(args),
        "run": {"qbits": q, "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                "l2": "flushed (256 MB write) between timed steps; W (400 MB) > L2",
                "multi_gpu": "each rank solves its own snapshot (seed + rank); value = per-round latency, max over ranks"},
        "replica_rounds_per_s": world / (t_step / 1e3),
        "pair_scores_per_s": n * m / (t_step / 1e3), "parity": parity,
        "roofline": {"bound": "hbm", "kernel": "ssp_rkey_kernel", "achieved": achieved, "peak": hbm,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "traffic_note": f"DRAM read+write bytes per launch (ncu --set full, profiles/{traffic_src})",
                     "algorithmic_bytes": dense_bytes, "kernel_ms": dense_ms,
                     "algorithmic_bytes_per_launch": dense_bytes / max(1.0, sum(x["dense_launches"] for x in stats_all) / len(stats_all)),
                     "note": "latency-bound: one cluster exchange per Dijkstra step (a step pops the minimum plus up to 2 tied warp minima); bytes = 4*m per pop",
                     "share_of_step": dense_ms / t_step},
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
        "gpu_launches": int(s["launches"]),
        "solver": dict({k: s[k] for k in ("levels", "par_steps", "dense_steps", "dense_searches", "dense_launches", "ms_dense",
                                          "ms_parallel", "row_scans", "total_q", "ms_match", "ms_canon", "canon_searches",
                                          "tight_edges", "dual_sweeps")},
                       dense_exchange_steps=s["rounds"],
                       us_per_pop=1e3 * s["ms_dense"] / max(1, s["dense_steps"]),
                       us_per_exchange_step=1e3 * s["ms_dense"] / max(1, s["rounds"]),
                       long_path_sms="8 (one 8-CTA cluster) for levels > 1300 columns, 1 below; scoring and parallel "
                                     "passes use all SMs"),
        "ms_match": auc_ms, "ms_per_step_all": times,
    }
    if sched_line is not None:
        line["schedule_drop_in"] = sched_line
    if mlp_line is not None:
        bf16 = bf16_peak()
        mlp_line.update({"peak_tflops": bf16, "frac": mlp_line["tflops"] / bf16, "bound": "tensor",
                         "tensor_frac_issued": mlp_line["tensor_tflops_issued"] / bf16})
        line["mlp_plugin"] = mlp_line
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        # CPU oracle port: rank 0 alone runs and prints; other ranks exit at once
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
