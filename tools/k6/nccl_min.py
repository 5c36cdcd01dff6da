"""Latency of one NCCL all-reduce(MIN) of a single int64 per step (the
per-pop exchange a NCCL-based K6 would need), one process per GPU.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/k6/nccl_min.py
"""
import json
import os
import time

import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
x = torch.full((1,), rank, dtype=torch.int64, device="cuda")
for _ in range(200):
    dist.all_reduce(x, op=dist.ReduceOp.MIN)
torch.cuda.synchronize()
dist.barrier()
res = {}
for n in (2000, 10000):
    t0 = time.perf_counter()
    for _ in range(n):
        dist.all_reduce(x, op=dist.ReduceOp.MIN)   # each depends on the previous (same buffer, one stream)
    torch.cuda.synchronize()
    res[n] = (time.perf_counter() - t0) / n * 1e6
t = torch.tensor([min(res.values())], dtype=torch.float64, device="cuda")
dist.all_reduce(t, op=dist.ReduceOp.MAX)
if rank == 0:
    print(json.dumps({"world": world, "us_per_allreduce_min_8B": float(t.item()),
                      "note": "back-to-back dependent all-reduces of one int64 on one stream, max over ranks"}))
dist.destroy_process_group()
