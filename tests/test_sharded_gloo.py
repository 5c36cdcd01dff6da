"""Multi-rank host logic of the row-sharded round on CPU (gloo, world size 2).

The GPU kernels are swapped for the oracle (scores) and the oracle Hungarian
(matching) so the sharding, gather and broadcast logic is exercised without a
GPU; the result must equal the single-process oracle round."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2303_13803_b200.sharded import shard_rows


def test_shard_rows_partition():
    for n in (0, 1, 7, 10, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_scorer(table, xs, ss, y, q):
    import torch
    from oracle import predictor_ref
    W = predictor_ref.predict_pairs_exact(table.axes, table.values, xs, ss, y)
    Q = np.rint(np.where(W >= 1e-6, W, 0.0) * 2.0 ** q).astype(np.int32)
    ldw = max(4, ((Q.shape[1] + 3) // 4) * 4)
    out = np.zeros((Q.shape[0], ldw), dtype=np.int32)
    out[:, : Q.shape[1]] = Q
    return torch.as_tensor(out)


def _oracle_matcher(W, n, m):
    import torch
    from oracle import matching_ref
    Q = W[:, :m].numpy().astype(np.int64)
    total, col = matching_ref.max_weight_total_int(Q)
    col = np.where((col < m) & (Q[np.arange(n), np.minimum(col, m - 1)] > 0), col, -1)
    return torch.as_tensor(col.astype(np.int32)), total


def _worker(rank, world, port, n, m, q):
    import torch.distributed as dist
    from paper_2303_13803_b200 import default_table
    from paper_2303_13803_b200.sharded import sharded_round
    from paper_2303_13803_b200.synth import make_cluster
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cl = make_cluster(n, m, seed=3)
        col, total = sharded_round(default_table(), cl.x, cl.share, cl.y, qbits=q,
                                   scorer=_oracle_scorer, matcher=_oracle_matcher)
        ref_col, ref_total = _oracle_matcher(_oracle_scorer(default_table(), cl.x, cl.share, cl.y, q), n, m)
        assert total == ref_total
        assert np.array_equal(col.numpy(), ref_col.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,m", [(37, 29), (40, 64)])
def test_sharded_round_gloo_world2(n, m):
    mp.spawn(_worker, args=(2, _free_port(), n, m, 20), nprocs=2, join=True)
