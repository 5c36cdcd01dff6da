"""Multi-GPU check of the row-sharded round (run under torchrun, NCCL):
every rank's col_of_row and total must equal a single-GPU round on rank 0."""
import os
import sys

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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
cl = make_cluster(n, n, seed=11)
t = default_table()
col, total = sharded_round(t, cl.x, cl.share, cl.y, qbits=20)
ref_col, ref_total = round_arrays(t, cl.x, cl.share, cl.y, qbits=20)
ok = total == ref_total and np.array_equal(col.cpu().numpy(), ref_col)
flag = torch.tensor([1 if ok else 0], device="cuda")
dist.all_reduce(flag, op=dist.ReduceOp.MIN)
if rank == 0:
    print(f"sharded_round world={dist.get_world_size()} n={n} total={total} ok={bool(flag.item())}")
dist.destroy_process_group()
sys.exit(0 if flag.item() else 1)
