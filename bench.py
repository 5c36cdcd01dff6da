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
region).  With N GPUs each rank solves its own replica (weak scaling, replicas
only in round 1 -- see DESIGN.md); timing is the max over ranks.

`--impl reference` times the CPU oracle port of the reference algorithm
(oracle/: scalar trilinear predict_point per pair + the O(n^3) Kuhn-Munkres)
on a bounded sample of the same workload and extrapolates to the metric's
10k x 10k round (the reference itself takes hours there).
"""

import argparse
import json
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
# CPU reference arm (oracle port of the reference algorithm)
# ---------------------------------------------------------------------------

def cpu_reference(n_target, m_target, seed, budget_s=20.0):
    """Time the oracle port on a bounded sample; extrapolate to n_target x m_target.

    predict: the scalar restatement of predictor.predict_point (the reference's
    per-pair loop body) timed on a sample of pairs -> per-pair cost x N*M.
    match:   the C restatement of matching._solve_min_assignment (O(n^3)) on a
             predictor-derived k x k sample -> cost x (n/k)^3.
    """
    from oracle import matching_ref, predictor_ref
    from paper_2303_13803_b200.synth import make_cluster
    t_axes = predictor_ref.DEFAULT_AXES
    vals = predictor_ref.default_table_values()
    k = 1024
    cl = make_cluster(k, k, seed=seed)
    # predict sample
    rng = np.random.default_rng(seed)
    npairs = 0
    us = rng.integers(0, k, 2000).tolist()
    vs = rng.integers(0, k, 2000).tolist()
    xs, ss, ys = cl.x.tolist(), cl.share.tolist(), cl.y.tolist()
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < min(3.0, budget_s / 4):
        for u, v in zip(us, vs):
            predictor_ref.predict_point(t_axes, vals, xs[u], ys[v], ss[u])
        npairs += 2000
    per_pair = (time.perf_counter() - t0) / npairs
    # match sample
    W = predictor_ref.predict_pairs_exact(t_axes, vals, cl.x, cl.share, cl.y)
    Wp = np.where(W >= 1e-6, W, 0.0)
    cost = Wp.max() - Wp
    t0 = time.perf_counter()
    matching_ref.solve_min_assignment(cost)
    t_match = time.perf_counter() - t0
    n_sq = max(n_target, m_target)
    est_s = per_pair * n_target * m_target + t_match * (n_sq / k) ** 3
    sample = (f"predict_point port timed on {npairs} pairs ({per_pair * 1e6:.2f} us/pair) x {n_target}*{m_target}; "
              f"C Kuhn-Munkres port on a {k}x{k} predictor-derived round ({t_match:.2f} s) x ({n_sq}/{k})^3; "
              f"1 thread; extrapolated to {n_target}x{m_target}")
    return est_s * 1e3, sample, t_match + per_pair * npairs


def ncu_traffic():
    """DRAM bytes per launch of ssp_cluster_kernel from the committed ncu capture."""
    for rnd in ("r01c", "r01b"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "ncu_cluster_traffic.json")) as f:
                return json.load(f)["dram_bytes_per_launch"], rnd
        except Exception:
            continue
    return None, None


def run_reference(args, rank, world):
    if rank != 0:
        return
    vals = []
    sample = ""
    for s in range(args.warmup + args.steps):
        ms, sample, _ = cpu_reference(args.n, args.m, args.seed + s, budget_s=10.0)
        if s >= args.warmup:
            vals.append(ms)
    v = float(np.mean(vals))
    line = {"metric": METRIC, "value": v, "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.n}x{args.m} scheduling round (predict + optimal match)",
                       "n_online": args.n, "n_offline": args.m},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "ms", "cores": 1, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "pair_scores_per_s": args.n * args.m / (v / 1e3)}
    print(json.dumps(line), flush=True)


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
        nat.check(lib.mux_score_table(ctx, tb, xd.data_ptr(), sd.data_ptr(), n, yd.data_ptr(), m,
                                      nat.MUX_SCORE_EXACT, nat.MUX_W_I32, q, Wq.data_ptr(), ldw, sptr))
        # the online / offline SM demands order rows and columns for the solver's warm start
        nat.check(lib.mux_match_keyed(ctx, Wq.data_ptr(), nat.MUX_W_I32, n, m, ldw, xd.data_ptr(), yd.data_ptr(),
                                      col.data_ptr(), 0, nat.ctypes.byref(total), nat.ctypes.byref(st), sptr))
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
        e2e = {"value": e2e_ms / world, "unit": "ms", "h2d_bytes_per_step": (2 * n + m) * 8 * world,
               "d2h_bytes_per_step": n * 4 * world, "per_round_ms": e2e_ms}

    # MLP plugin (tcgen05) scoring of the same N x M pairs: tensor-core roofline
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
        mlp_line = {"ms": mlp_ms, "tflops": flops / (mlp_ms / 1e3) / 1e12, "flops": flops,
                    "note": "layers 2-3 as tcgen05 kind::f16 M128xN64xK16, fp32 TMEM accumulate"}

    if rank != 0:
        return
    hbm, peak_kind = peaks()
    # dominant kernel: ssp_cluster_kernel (csrc/ssp.cu), the thread-block-cluster
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
        cpu_ms, sample, _ = cpu_reference(n, m, args.seed)
        cpu = {"value": cpu_ms, "unit": "ms", "cores": 1, "kind": "port", "sample": sample}
    s = stats_all[-1]
    value = t_step / world
    line = {
        "metric": METRIC, "value": value, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32 (f64 scoring)", "data": "synthetic",
        "config": {"workload": f"{n}x{m} scheduling round (predict + optimal match), replicas per GPU",
                   "n_online": n, "n_offline": m, "qbits": q, "parallelism": f"replicas x{world}",
                   "l2": "flushed (256 MB write) between timed steps; W (400 MB) > L2"},
        "pair_scores_per_s": n * m * world / (t_step / 1e3),
        "roofline": {"bound": "hbm", "kernel": "ssp_cluster_kernel", "achieved": achieved, "peak": hbm,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "traffic_note": f"DRAM read+write bytes per launch (ncu --set full, profiles/{traffic_src})",
                     "algorithmic_bytes": dense_bytes, "kernel_ms": dense_ms,
                     "algorithmic_bytes_per_launch": dense_bytes / max(1.0, sum(x["dense_launches"] for x in stats_all) / len(stats_all)),
                     "note": "latency-bound: one dependent pop per step (sequential Dijkstra); bytes = 4*m per pop",
                     "share_of_step": dense_ms / t_step},
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
        "gpu_launches": int(s["launches"]) + 3,
        "solver": {k: s[k] for k in ("levels", "par_steps", "dense_steps", "dense_searches", "dense_launches", "ms_dense", "ms_parallel",
                                     "row_scans", "total_q", "ms_match", "ms_canon", "canon_searches", "tight_edges",
                                     "dual_sweeps")},
        "ms_match": auc_ms, "ms_per_step_all": times,
    }
    if mlp_line is not None:
        bf16 = bf16_peak()
        mlp_line.update({"peak_tflops": bf16, "frac": mlp_line["tflops"] / bf16, "bound": "tensor"})
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
