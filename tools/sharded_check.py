"""Multi-GPU row-sharded round (run under torchrun, NCCL): stripes scored
straight into the root's HBM over NVLink (sharded.py, transport="p2p"), the
exact matching on the root.  Every rank's col_of_row and total must equal a
single-GPU round; prints the root's phase times (JSON).

    torchrun --nproc-per-node N tools/sharded_check.py [n] [reps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from paper_2303_13803_b200 import default_table, round_arrays
from paper_2303_13803_b200.sharded import sharded_round
from paper_2303_13803_b200.synth import make_cluster

rank = int(os.environ["RANK"])
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cl = make_cluster(n, n, seed=11)
t = default_table()
res = []
for r in range(reps + 1):
    tim = {}
    dist.barrier()
    t0 = time.perf_counter()
    col, total = sharded_round(t, cl.x, cl.share, cl.y, qbits=30, timings=tim)
    tim["round_ms"] = (time.perf_counter() - t0) * 1e3
    if r > 0:
        res.append(tim)
ref_col, ref_total = round_arrays(t, cl.x, cl.share, cl.y, qbits=30)
ok = total == ref_total and np.array_equal(col.cpu().numpy(), ref_col)
flag = torch.tensor([1 if ok else 0], device="cuda")
dist.all_reduce(flag, op=dist.ReduceOp.MIN)
sc = torch.tensor([max(x["score_ms"] for x in res)], device="cuda", dtype=torch.float64)
dist.all_reduce(sc, op=dist.ReduceOp.MAX)
if rank == 0:
    med = lambda k: sorted(x[k] for x in res)[len(res) // 2]
    print(json.dumps({"world": dist.get_world_size(), "n": n, "total": total, "identical_to_1gpu": bool(flag.item()),
                      "transport": "p2p (scoring kernel stores into the root's HBM over NVLink)",
                      "score_ms_median": med("score_ms"), "score_ms_max_over_ranks": float(sc.item()),
                      "match_ms_median": med("match_ms"), "round_ms_median": med("round_ms"),
                      "bytes_written_remote_per_rank": 4 * n * ((n + 3) // 4 * 4) // dist.get_world_size()}))
dist.destroy_process_group()
sys.exit(0 if flag.item() else 1)
