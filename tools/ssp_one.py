"""One n x n round (exact scoring + solve) through mux_round_dev, for timing
and ncu captures: python tools/ssp_one.py [n] [repeats]."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_13803_b200 import _native as nat, default_table
from paper_2303_13803_b200.synth import make_cluster
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
q = int(os.environ.get("QBITS", "30"))
t = default_table(); tb, keep = nat.table_struct(t.axes, t.values)
cl = make_cluster(n, n, seed=int(os.environ.get("SEED", "0")))
dev = torch.device("cuda", 0)
xd, sd, yd = (torch.as_tensor(a, device=dev) for a in (cl.x, cl.share, cl.y))
ldw = (n + 3) // 4 * 4
Wq = torch.empty((n, ldw), dtype=torch.int32, device=dev)
col = torch.empty(n, dtype=torch.int32, device=dev)
lib, ctx = nat.load(), nat.context(0)
tot, st = nat.ctypes.c_int64(0), nat.MuxStats()
sp = nat.ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nat.check(lib.mux_round_dev(ctx, tb, xd.data_ptr(), sd.data_ptr(), n, yd.data_ptr(), n, q, Wq.data_ptr(), ldw,
                                col.data_ptr(), None, None, 0, nat.ctypes.byref(tot), nat.ctypes.byref(st), sp))
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    d = st.as_dict()
    print(f"round {r}: {ms:.2f} ms total {tot.value} dense {d['ms_dense']:.2f} ms pops {d['dense_steps']} "
          f"us/pop {1e3 * d['ms_dense'] / max(1, d['dense_steps']):.3f} steps {d['rounds']} "
          f"us/step {1e3 * d['ms_dense'] / max(1, d['rounds']):.3f} parallel {d['ms_parallel']:.2f} canon {d['ms_canon']:.2f}",
          flush=True)
