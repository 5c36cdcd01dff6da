"""Multi-GPU scheduling round: row-sharded scoring written straight into the
root's HBM over NVLink, one exact matching on the root.

One process per GPU (`torch.distributed`).  Pair scoring is row-independent
(north_star: "pair scoring is row-sharded with no communication"): rank r
scores its contiguous stripe of online rows.  With `transport="p2p"` (the
default on GPUs) the root exports its weight buffer through a CUDA IPC
handle, every rank maps it (peer access over NVLink 5) and the scoring
kernel's stores land in the root's HBM directly -- no gather, no staging
copy; a barrier then hands the complete matrix to the root's solver.
`transport="gather"` collects the stripes with a collective instead (the
host-logic path the CPU/gloo tests exercise).

Why the matching itself is not sharded (SURVEY.md §8e's K6): its critical
path is a chain of dependent Dijkstra pops (~1.2 us each on one GPU, 8 SMs
of a thread-block cluster).  Splitting the columns across GPUs adds an
all-GPU minimum per pop: measured 2.9 / 6.6 us for a peer-memory exchange among
2 / 4 GPUs and 21 us for an NCCL all-reduce of one int64
(profiles/r02/k6_*.json), i.e. every pop would get 3-18x slower.  The solve
therefore stays on one GPU; `bench.py --gpus N` measures replicas (N
snapshots, weak scaling) and reports this sharded round beside it.
"""

import ctypes

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


class PeerMatrix:
    """The root's int32 weight buffer [n, ldw], mapped into every rank."""

    def __init__(self, n, ldw, group=None, root=0):
        import torch
        import torch.distributed as dist
        from . import _native as nat
        self.n, self.ldw = n, ldw
        rank = dist.get_rank(group)
        dev = torch.device("cuda", torch.cuda.current_device())
        lib, ctx = nat.load(), nat.context()
        handle = torch.zeros(64, dtype=torch.uint8, device=dev)
        ptr = ctypes.c_void_p()
        if rank == root:
            h = (ctypes.c_ubyte * 64)()
            nat.check(lib.mux_ipc_export(ctx, 4 * n * ldw, ctypes.byref(ptr), h))
            handle.copy_(torch.as_tensor(np.frombuffer(bytes(h), dtype=np.uint8).copy()))
        dist.broadcast(handle, src=root, group=group)
        if rank != root:
            hb = (ctypes.c_ubyte * 64).from_buffer_copy(handle.cpu().numpy().tobytes())
            nat.check(lib.mux_ipc_import(ctx, hb, ctypes.byref(ptr)))
        self.ptr = ptr.value

    def rows(self, start):
        return self.ptr + 4 * start * self.ldw


def sharded_round(table, x, share, y, qbits=30, group=None, root=0, scorer=None, matcher=None,
                  transport=None, timings=None):
    """One round across the ranks of `group`; every rank returns col_of_row.

    transport "p2p" (GPU default): stripes scored straight into the root's
    buffer over NVLink.  "gather": `scorer(table, x_stripe, share_stripe, y,
    qbits)` -> int tensor [rows, ldw] per rank, gathered to the root, then
    `matcher(W, n, m)` -> (col int32 tensor, total) (defaults: the CUDA
    kernels).  `timings` (dict) receives the root-side phase times in ms.
    """
    import time
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n, m = len(x), len(y)
    if transport is None:
        transport = "gather" if (scorer is not None or not torch.cuda.is_available()) else "p2p"
    s, e = shard_rows(n, world, rank)
    t0 = time.perf_counter()
    if transport == "p2p":
        from . import _native as nat
        from .predictor import _as_table_arrays
        dev = torch.device("cuda", torch.cuda.current_device())
        ldw = max(4, (m + 3) // 4 * 4)
        pm = PeerMatrix(n, ldw, group=group, root=root)
        axes, vals = _as_table_arrays(table)
        tb, keep = nat.table_struct(axes, vals)
        xs, ss, yy = (torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
                      for a in (np.asarray(x)[s:e], np.asarray(share)[s:e], np.asarray(y)))
        dist.barrier(group=group)
        t1 = time.perf_counter()
        if e > s:
            nat.check(nat.load().mux_score_table(nat.context(), tb, xs.data_ptr(), ss.data_ptr(), e - s, yy.data_ptr(),
                                                 m, nat.MUX_SCORE_EXACT, nat.MUX_W_I32, qbits, pm.rows(s), ldw,
                                                 nat.stream_ptr()))
        torch.cuda.synchronize()
        dist.barrier(group=group)        # every stripe is in the root's HBM
        t2 = time.perf_counter()
        col = torch.empty(n, dtype=torch.int32, device=dev)
        total = torch.zeros(1, dtype=torch.int64, device=dev)
        if rank == root:
            from .matching import match_dense_ptr
            c, tq = match_dense_ptr(pm.ptr, n, m, ldw, np.asarray(x), np.asarray(y))
            col.copy_(c)
            total.fill_(int(tq))
        t3 = time.perf_counter()
        del keep
        if timings is not None:
            timings.update(setup_ms=(t1 - t0) * 1e3, score_ms=(t2 - t1) * 1e3, match_ms=(t3 - t2) * 1e3)
    else:
        if scorer is None:
            from .predictor import predict_pairs

            def scorer(t, xs, ss, yy, q):
                return predict_pairs(t, xs, ss, yy, dtype="int32", qbits=q).contiguous()
        if matcher is None:
            from .matching import match_dense
            matcher = match_dense
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
