"""One 10k x 10k scoring + solve through the C ABI (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_13803_b200 import _native as nat, default_table
from paper_2303_13803_b200.synth import make_cluster
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
q = 30
t = default_table(); tb, keep = nat.table_struct(t.axes, t.values)
cl = make_cluster(n, n, seed=0)
dev = torch.device("cuda", 0)
xd, sd, yd = (torch.as_tensor(a, device=dev) for a in (cl.x, cl.share, cl.y))
ldw = (n + 3) // 4 * 4
Wq = torch.empty((n, ldw), dtype=torch.int32, device=dev)
col = torch.empty(n, dtype=torch.int32, device=dev)
lib, ctx = nat.load(), nat.context(0)
tot, st = nat.ctypes.c_int64(0), nat.MuxStats()
sp = nat.ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
nat.check(lib.mux_score_table(ctx, tb, xd.data_ptr(), sd.data_ptr(), n, yd.data_ptr(), n, nat.MUX_SCORE_EXACT,
                              nat.MUX_W_I32, q, Wq.data_ptr(), ldw, sp))
nat.check(lib.mux_match_keyed(ctx, Wq.data_ptr(), nat.MUX_W_I32, n, n, ldw, xd.data_ptr(), yd.data_ptr(),
                              col.data_ptr(), 0, nat.ctypes.byref(tot), nat.ctypes.byref(st), sp))
torch.cuda.synchronize()
print("total", tot.value, {k: v for k, v in st.as_dict().items() if k in ("levels", "par_steps", "dense_steps", "ms_dense", "ms_parallel", "ms_match")})
