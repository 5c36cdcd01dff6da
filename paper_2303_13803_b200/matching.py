"""Maximum-weight bipartite matching on the GPU.

Mirrors /root/reference/pkg/src/muxsim/matching.py.  `max_weight_matching`
keeps the reference's contract (sorted ids, zero padding to square, the 1e-6
weight floor, only W > 0 pairs emitted, total summed in row order) but solves
with libmuxflow's multilevel shortest-path solver (csrc/ssp.cu) on integer
weights rint(w * 2^qbits), followed by the reference's tie canonicalisation
(csrc/canon.cu).  Dyadic inputs with granularity >= 2^-qbits (all of the
reference's tests) are solved exactly; general floats are solved exactly for
their quantisation (an optimum of the quantised problem is within
n * 2^-(qbits+1) of the float optimum).  `match_dense` / `match_dense_ptr`
are the array-level entries the scheduling round and the benchmarks use.
"""

import math
import random
from dataclasses import dataclass, field
from typing import Dict, List, Tuple

import numpy as np

from . import _native as nat

WEIGHT_FLOOR = 1e-6


@dataclass(frozen=True)
class BipartiteGraph:
    left: Tuple[str, ...]
    right: Tuple[str, ...]
    weights: Dict[Tuple[str, str], float] = field(default_factory=dict)

    def __post_init__(self):
        lset, rset = set(self.left), set(self.right)
        if len(lset) != len(self.left) or len(rset) != len(self.right):
            raise ValueError("duplicate node ids in bipartite graph")
        for (l, r), w in self.weights.items():
            if l not in lset or r not in rset:
                raise ValueError(f"edge ({l!r}, {r!r}) references unknown node")
            if not math.isfinite(w):
                raise ValueError(f"edge ({l!r}, {r!r}) has non-finite weight {w}")


@dataclass(frozen=True)
class Matching:
    pairs: Tuple[Tuple[str, str], ...]
    total_weight: float


def max_qbits(n: int, cap: int = 30) -> int:
    """Largest quantisation (<= `cap` bits; int32 storage up to 30) whose
    auction prices fit the 64-bit bid packing for an n x n problem."""
    idbits = max(1, int(n).bit_length())
    q = int(math.floor(60 - idbits - math.log2(n + 1))) - 1
    return max(1, min(int(cap), q))


def round_qbits(n: int) -> int:
    """Quantisation of a scheduling round: the exact-parity mode (int64
    weights, 40 bits) for rounds up to 6,144 on the larger
    side, else 30-bit int32 weights (the int64 matrix of a large round doubles
    the bytes every long-path pop loads).  Both run on the multilevel
    shortest-path solver (csrc/ssp.cu, csrc/ssp_w64.cu)."""
    return 40 if n <= 6144 else 30


def match_dense(Wq, n=None, m=None, stats=False):
    """Optimal max-weight matching of a non-negative integer weight tensor.

    Wq: CUDA torch tensor [N, ldw] (int32 or int64, row stride multiple of 16
    bytes); n/m default to its shape.  Returns (col_of_row int32 CUDA tensor
    [N] with -1 for unmatched rows, total_q int[, stats dict]).
    """
    torch = nat.torch_cuda()
    if Wq.dim() != 2:
        raise ValueError("Wq must be 2-D")
    N = Wq.shape[0] if n is None else int(n)
    M = Wq.shape[1] if m is None else int(m)
    wtype = {torch.int32: nat.MUX_W_I32, torch.int64: nat.MUX_W_I64}.get(Wq.dtype)
    if wtype is None:
        raise ValueError("Wq must be int32 or int64")
    if Wq.stride(1) != 1:
        raise ValueError("Wq rows must be contiguous")
    col = torch.empty(max(N, 1), dtype=torch.int32, device=Wq.device)
    total = nat.ctypes.c_int64(0)
    st = nat.MuxStats()
    nat.check(nat.load().mux_match(nat.context(Wq.device.index), Wq.data_ptr(), wtype, N, M, Wq.stride(0),
                                   col.data_ptr(), 0, nat.ctypes.byref(total), nat.ctypes.byref(st),
                                   nat.stream_ptr(Wq.device)))
    if stats:
        return col[:N], int(total.value), st.as_dict()
    return col[:N], int(total.value)


def match_dense_ptr(w_ptr, n, m, ldw, rowkey=None, colkey=None):
    """match_dense on a raw device int32 buffer [n][ldw] (e.g. the root's
    peer-written weight matrix, sharded.PeerMatrix), optionally ordered by
    host keys (the online / offline SM demands).  Returns (col int32 CUDA
    tensor [n], total_q)."""
    torch = nat.torch_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    col = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    total = nat.ctypes.c_int64(0)
    st = nat.MuxStats()
    rk = ck = None
    if rowkey is not None and colkey is not None:
        rk = torch.as_tensor(np.ascontiguousarray(rowkey, dtype=np.float64), device=dev)
        ck = torch.as_tensor(np.ascontiguousarray(colkey, dtype=np.float64), device=dev)
    nat.check(nat.load().mux_match_keyed(nat.context(), w_ptr, nat.MUX_W_I32, n, m, ldw,
                                         rk.data_ptr() if rk is not None else None,
                                         ck.data_ptr() if ck is not None else None, col.data_ptr(), 0,
                                         nat.ctypes.byref(total), nat.ctypes.byref(st), nat.stream_ptr()))
    return col[:n], int(total.value)


def quantise(W, qbits):
    """Reference edge rule (w < 1e-6 -> missing) then rint(w * 2^qbits)."""
    W = np.asarray(W, dtype=np.float64)
    Wf = np.where(W >= WEIGHT_FLOOR, W, 0.0)
    return np.rint(Wf * float(2 ** qbits)).astype(np.int64)


def max_weight_matching(g: BipartiteGraph, qbits: int = None) -> Matching:
    """Optimal maximum-weight matching (matching.py:148-208), solved on the GPU."""
    torch = nat.torch_cuda()
    L = sorted(g.left)
    R = sorted(g.right)
    nl, nr = len(L), len(R)
    if max(nl, nr) == 0:
        return Matching(pairs=(), total_weight=0.0)
    li = {l: i for i, l in enumerate(L)}
    ri = {r: j for j, r in enumerate(R)}
    W = np.zeros((nl, nr))
    for (l, r), w in g.weights.items():
        if w >= WEIGHT_FLOOR:
            W[li[l], ri[r]] = w
    if nl == 0 or nr == 0:
        return Matching(pairs=(), total_weight=0.0)
    if qbits is None:
        # resolution 2^-q with every rint(w * 2^q) inside int32 and the bid packing
        wmax = float(W.max())
        q = max_qbits(max(nl, nr))
        if wmax > 0:
            q_int = int(math.floor(math.log2((2 ** 31 - 1) / wmax)))
            q_pack = q - max(0, int(math.ceil(math.log2(wmax))))
            q = max(1, min(q_int, q_pack))
    else:
        q = int(qbits)
    Q = quantise(W, q)
    ldw = ((nr + 3) // 4) * 4
    Qp = np.zeros((nl, ldw), dtype=np.int32)
    Qp[:, :nr] = Q
    dev = torch.device("cuda", torch.cuda.current_device())
    col, _total = match_dense(torch.as_tensor(Qp, device=dev), nl, nr)
    col = col.cpu().numpy()
    pairs = []
    total = 0.0
    for i in range(nl):
        j = int(col[i])
        if j >= 0 and W[i, j] > 0.0:
            pairs.append((L[i], R[j]))
            total += float(W[i, j])
    return Matching(pairs=tuple(pairs), total_weight=total)


def random_maximal_matching(g: BipartiteGraph, rng: random.Random) -> Matching:
    """Seeded random maximal matching over present edges: the reference's
    `muxflow_random_match` ablation baseline (matching.py:211-231); host-only,
    it is not on the matching hot path."""
    order = sorted(g.left)
    rng.shuffle(order)
    adj: Dict[str, List[Tuple[str, float]]] = {l: [] for l in g.left}
    for (l, r), w in sorted(g.weights.items()):
        if w >= WEIGHT_FLOOR:
            adj[l].append((r, w))
    taken, chosen, total = set(), [], 0.0
    for l in order:
        avail = [(r, w) for r, w in adj[l] if r not in taken]
        if not avail:
            continue
        r, w = avail[rng.randrange(len(avail))]
        taken.add(r)
        chosen.append((l, r))
        total += w
    chosen.sort()
    return Matching(pairs=tuple(chosen), total_weight=total)
