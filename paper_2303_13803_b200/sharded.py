"""Multi-GPU scheduling round: row-sharded scoring, one auction.

One process per GPU (`torch.distributed`, NCCL over NVLink).  Pair scoring is
row-independent, so each rank scores its contiguous stripe of online rows
with no communication (north_star: "pair scoring is row-sharded with no
communication").  The stripes are then gathered to the root rank, which runs
the auction on the full matrix and broadcasts col_of_row.

Why the matching is not sharded: the auction's critical path is a chain of
dependent bids (Jacobi rounds plus a Gauss-Seidel tail);
at 10k x 10k a per-round collective (~10 us) times ~10^4 rounds exceeds the
whole single-GPU solve, and the tail is sequential.  `bench.py --gpus N`
therefore measures replicas (N independent snapshots, weak scaling) and this
module provides the row-sharded round for snapshots whose scoring dominates.
"""

import numpy as np


def shard_rows(n: int, world: int, rank: int):
    """Contiguous [start, end) of n rows for `rank` of `world` (sizes differ by <= 1)."""
    base, rem = divmod(int(n), int(world))
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def gather_stripes(stripe, n, world, rank, group=None, root=0):
    """Assemble the [n, ldw] matrix on `root` from per-rank stripes [rows_r, ldw].

    Stripes are padded to the largest shard so the collective sees equal
    sizes; returns the full matrix on root and None elsewhere.
    """
    import torch
    import torch.distributed as dist
    rows_max = shard_rows(n, world, 0)[1] - shard_rows(n, world, 0)[0]
    ldw = stripe.shape[1]
    padded = torch.zeros((rows_max, ldw), dtype=stripe.dtype, device=stripe.device)
    padded[: stripe.shape[0]] = stripe
    parts = [torch.empty_like(padded) for _ in range(world)] if rank == root else None
    dist.gather(padded, parts, dst=root, group=group)
    if rank != root:
        return None
    full = torch.empty((n, ldw), dtype=stripe.dtype, device=stripe.device)
    for r in range(world):
        s, e = shard_rows(n, world, r)
        full[s:e] = parts[r][: e - s]
    return full


def sharded_round(table, x, share, y, qbits=20, group=None, root=0, scorer=None, matcher=None):
    """One round across the ranks of `group`; every rank returns col_of_row.

    `scorer(table, x_stripe, share_stripe, y, qbits)` -> int tensor [rows, ldw]
    and `matcher(W, n, m)` -> (col int32 tensor, total) default to the CUDA
    kernels (predict_pairs / match_dense).
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n, m = len(x), len(y)
    if scorer is None:
        from .predictor import predict_pairs

        def scorer(t, xs, ss, yy, q):
            return predict_pairs(t, xs, ss, yy, dtype="int32", qbits=q).contiguous()
    if matcher is None:
        from .matching import match_dense
        matcher = match_dense
    s, e = shard_rows(n, world, rank)
    stripe = scorer(table, np.asarray(x)[s:e], np.asarray(share)[s:e], np.asarray(y), qbits)
    full = gather_stripes(stripe, n, world, rank, group=group, root=root)
    col = torch.empty(n, dtype=torch.int32, device=stripe.device)
    total = torch.zeros(1, dtype=torch.int64, device=stripe.device)
    if rank == root:
        c, t = matcher(full, n, m)
        col.copy_(c)
        total.fill_(int(t))
    dist.broadcast(col, src=root, group=group)
    dist.broadcast(total, src=root, group=group)
    return col, int(total.item())
