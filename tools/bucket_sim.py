"""Analysis: how many synchronised rounds would a bucketed (label-correcting)
long search need, against the one-pop-per-exchange Dijkstra of
ssp_rkey_kernel?  Reads the level dumps MUX_SSP_DUMP writes (header
{m, nreal, ndef, level, wsize}, A, p, roc, cor, defer) and, per deferred row
in order: runs the exact Dijkstra (pops, path hops), simulates the bucketed
variants on the same state (rounds, relaxed rows, same D), then applies the
Dijkstra result so the next row starts from the kernel's state.

    python tools/bucket_sim.py DUMPDIR
"""

import glob
import os
import sys

import numpy as np
import torch

INF = 1 << 62


def load(path):
    with open(path, "rb") as f:
        m, nreal, ndef, level, ws = np.frombuffer(f.read(20), dtype=np.int32)
        a = np.frombuffer(f.read(ws * nreal * m), dtype=np.int32 if ws == 4 else np.int64).reshape(nreal, m)
        p = np.frombuffer(f.read(8 * m), dtype=np.int64)
        roc = np.frombuffer(f.read(4 * m), dtype=np.int32)
        cor = np.frombuffer(f.read(4 * m), dtype=np.int32)
        de = np.frombuffer(f.read(4 * ndef), dtype=np.int32)
    return int(m), int(nreal), int(level), a, p, roc, cor, de


def dijkstra(A, p, roc, s, dev):
    m = p.numel()
    d = p - A[s] + (A[s] - p).max()
    pred = torch.full((m,), s, dtype=torch.int64, device=dev)
    done = torch.zeros(m, dtype=torch.bool, device=dev)
    free = roc < 0
    idx = torch.arange(m, device=dev)
    pops = 0
    while True:
        key = torch.where(done, INF, d * 2 * m + (~free).long() * m + idx)
        j = int(key.argmin())
        if bool(free[j]):
            return d, pred, done, j, int(d[j]), pops
        pops += 1
        done[j] = True
        i = int(roc[j])
        base = d[j] + A[i, j] - p[j]
        nd = base + p - A[i]
        upd = (nd < d) & ~done
        d = torch.where(upd, nd, d)
        pred = torch.where(upd, torch.full_like(pred, i), pred)


def bucketed(A, p, roc, s, dev, rule, arg):
    m = p.numel()
    d = p - A[s] + (A[s] - p).max()
    sd = torch.full((m,), INF, dtype=torch.int64, device=dev)   # value a column was relaxed at
    free = roc < 0
    rounds = rows = 0
    while True:
        D = int(torch.where(free, d, INF).min())
        U = (~free) & (d < sd) & (d < D)
        if not bool(U.any()):
            return D, rounds, rows
        du = torch.where(U, d, INF)
        mu = int(du.min())
        if rule == "delta":
            th = mu + arg
        else:   # k smallest
            k = min(arg, int(U.sum()))
            th = int(torch.kthvalue(du[U], k).values)
        F = U & (d <= th)
        cols = F.nonzero().squeeze(1)
        rows_i = roc[cols].long()
        base = d[cols] + A[rows_i, cols] - p[cols]
        nd = (base[:, None] + p[None, :] - A[rows_i]).min(0).values
        sd[cols] = d[cols]
        d = torch.minimum(d, nd)
        rounds += 1
        rows += cols.numel()


def main(dump_dir):
    dev = torch.device("cuda")
    rules = [("delta", 0), ("delta", 1 << 12), ("delta", 1 << 16), ("delta", 1 << 20), ("delta", 1 << 24),
             ("k", 4), ("k", 16), ("k", 64)]
    tot = {"pops": 0, "hops": 0, **{f"{r}{a}": [0, 0] for r, a in rules}}
    for path in sorted(glob.glob(os.path.join(dump_dir, "lvl*.bin")), key=os.path.getmtime):
        m, nreal, level, a, p, roc, cor, de = load(path)
        A = torch.zeros((m, m), dtype=torch.int64, device=dev)
        A[:nreal] = torch.as_tensor(a.astype(np.int64), device=dev)
        p = torch.as_tensor(p.copy(), device=dev)
        roc = torch.as_tensor(roc.astype(np.int64), device=dev)
        cor = torch.as_tensor(cor.astype(np.int64), device=dev)
        for s in de.tolist():
            d, pred, done, jf, D, pops = dijkstra(A, p, roc, s, dev)
            line = [f"{os.path.basename(path)} m {m} row {s}: pops {pops}"]
            for r, arg in rules:
                Db, rounds, rows = bucketed(A, p, roc, s, dev, r, arg)
                assert Db == D, (r, arg, Db, D)
                tot[f"{r}{arg}"][0] += rounds
                tot[f"{r}{arg}"][1] += rows
                line.append(f"{r}{arg}: {rounds} rounds {rows} rows")
            # apply the Dijkstra result (the kernel's state for the next row)
            p = torch.where(done, p + (D - d), p)
            j, hops = jf, 0
            while True:
                i = int(pred[j])
                jn = int(cor[i]) if i != s else -1
                roc[j] = i
                cor[i] = j
                hops += 1
                if i == s:
                    break
                j = jn
            line.insert(1, f"hops {hops}")
            tot["pops"] += pops
            tot["hops"] += hops
            print(" | ".join(line), flush=True)
    print("TOTAL", tot)


if __name__ == "__main__":
    main(sys.argv[1])
