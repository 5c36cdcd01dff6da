"""Config-5 trace replay on the GPU round (BASELINE.json config 5; SURVEY.md
§8 row f3).

The reference runs one scheduling round every `SchedulerConfig.interval`
seconds from its event engine (`_Engine._on_round`,
/root/reference/pkg/src/muxsim/simengine.py:665-735): rows are the healthy
onlines with their `dynamic_sm` share at t, columns the offline jobs that
may be (re)placed.  This replays 100 such rounds of the reference's own
`gen_trace({"gpus": 10000, "horizon_s": 90000, "offline":
{"count_per_gpu": 4.0}}, seed=0)` (generated once on the build box into
tests/golden/replay_cfg5.npz, see tests/golden/make_replay_fixture.py):
round k at t = (k + 1) * 900 s, rows = onlines with share > 0 (peak SM
activity of the trailing window, share from `dynamic_sm`), columns = jobs
submitted by t within the memory quota (0 -> 40k over the first 12 hours).

Each round is one `mux_round_dev` call on HBM-resident features.  With
`warm=True` the previous round's optimal column prices are carried to the
columns that persist and its placements that are still tight under them are
kept (new columns are priced by the c-transform of the row profits), which
replaces the multilevel warm start of the solver: only the rows whose
features changed (~11 % per round in this trace) are searched.  The optimum
is the same either way (the dual certificate and the CPU totals check it),
only the work changes.
"""

import os
import time

import numpy as np

from . import _native as nat
from .tables import default_table

FIXTURE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                       "replay_cfg5.npz")
MEM_QUOTA = 0.40


class Replay:
    def __init__(self, path=FIXTURE):
        fx = np.load(path)
        self.levels = fx["levels"]
        self.lvl = fx["lvl"]
        self.share_q = fx["share_q"]
        self.y_all = fx["y"]
        self.mem = fx["mem"]
        self.submit = fx["submit"]
        self.interval = float(fx["interval"])
        self.quantum = float(fx["quantum"])
        self.rounds = self.lvl.shape[0]

    def round(self, k):
        """(x, share, y, row ids, column ids) of round k."""
        n = self.levels.shape[0]
        x = self.levels[np.arange(n), self.lvl[k]]
        share = self.share_q[k].astype(np.float64) * self.quantum   # quantize_share's floor(.) * quantum
        rows = np.nonzero(share > 0.0)[0]
        t = (k + 1) * self.interval
        cols = np.nonzero((self.submit <= t) & (self.mem <= MEM_QUOTA))[0]
        return x[rows], share[rows], self.y_all[cols], rows, cols


def run(rounds=100, qbits=30, warm=True, path=FIXTURE, device=0, on_round=None):
    """Replay `rounds` rounds; returns a list of per-round dicts (n, m, ms
    device time of the round, total_q, warm, stats)."""
    torch = nat.torch_cuda()
    rp = Replay(path)
    dev = torch.device("cuda", device)
    lib, ctx = nat.load(), nat.context(device)
    t = default_table()
    tb, keep = nat.table_struct(t.axes, t.values)
    stream = torch.cuda.current_stream(dev)
    sptr = nat.ctypes.c_void_p(stream.cuda_stream)
    njobs = rp.y_all.shape[0]
    carried = np.full(njobs, np.iinfo(np.int64).min, dtype=np.int64)
    job_of_online = np.full(rp.levels.shape[0], -1, dtype=np.int64)   # previous round's placement
    out = []
    for k in range(min(rounds, rp.rounds)):
        x, s, y, rows, cols = rp.round(k)
        n, m = x.shape[0], y.shape[0]
        pin = carried[cols]
        known = float(np.mean(pin != np.iinfo(np.int64).min)) if m else 0.0
        use_warm = bool(warm and n <= m and known >= 0.5)
        pos_of_job = np.full(njobs, -1, dtype=np.int64)
        pos_of_job[cols] = np.arange(m)
        prev = job_of_online[rows]
        wcol = np.where(prev >= 0, pos_of_job[np.maximum(prev, 0)], -1).astype(np.int32)
        xd, sd, yd = (torch.as_tensor(a, device=dev) for a in (x, s, y))
        ldw = max(4, (m + 3) // 4 * 4)
        Wq = torch.empty((n, ldw), dtype=torch.int32, device=dev)
        col = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        prices = torch.as_tensor(pin if m else np.zeros(1, dtype=np.int64), device=dev)
        wcol_d = torch.as_tensor(wcol if n else np.zeros(1, dtype=np.int32), device=dev)
        tot, st = nat.ctypes.c_int64(0), nat.MuxStats()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0.record(stream)
        nat.check(lib.mux_round_dev(ctx, tb, xd.data_ptr(), sd.data_ptr(), n, yd.data_ptr(), m, qbits,
                                    Wq.data_ptr(), ldw, col.data_ptr(), prices.data_ptr(), wcol_d.data_ptr(),
                                    1 if use_warm else 0,
                                    nat.ctypes.byref(tot), nat.ctypes.byref(st), sptr))
        e1.record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - w0) * 1e3
        pout = prices.cpu().numpy()[:m]
        carried[cols] = pout
        c = col.cpu().numpy()[:n].astype(np.int64)
        job_of_online[:] = -1
        job_of_online[rows] = np.where(c >= 0, cols[np.maximum(c, 0)], -1)
        rec = {"round": k, "n": n, "m": m, "ms": e0.elapsed_time(e1), "wall_ms": wall, "total_q": int(tot.value),
               "warm": use_warm, "stats": st.as_dict()}
        if on_round is not None:
            on_round(rec, Wq[:, :m], col[:n])
        out.append(rec)
    del keep
    return out
