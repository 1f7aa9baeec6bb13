"""Cross-GPU sharding of one zip-up, host logic on CPU with gloo,
world size 2: the column-shard partition, the R-tree exchange (all-gather of each shard's m x m
factor; the R of the stacked factors is the R of T^H) and the carry exchange (all-gather of
the carry slabs U_k^T T_t, reassembled into the next site's carry) -- driven by the same
ShardExchange the GPU path uses.  The per-shard arithmetic here is a NumPy mirror of the
library's steps (test code); the sharded result must equal the unsharded oracle zip-up."""
import math
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_20226_b200 import gen
from paper_2602_20226_b200.shard import ShardExchange, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    p = gen.cfg3(L=9, R=12, max_rank=10, eps=1e-6)
    return p.kind, p.op.cores, p.x.cores, p.eps, p.max_rank


def sharded_numpy(kind, op, x, eps, max_rank, ex, S, rank, ls):
    """NumPy mirror of large.cu large_zipup_sharded (one process's part), exchanging through ex."""
    from oracle.tt import right_orthonormalize, tail_sum, truncation_rank
    from oracle.zipup import site_matrix
    X = right_orthonormalize(x)
    O = right_orthonormalize(op) if op is not None else None
    L = len(X)
    G = np.ones((1, 1, 1))
    mcap = int(math.isqrt(ex.r_elems))
    cores, ranks, delta2 = [], [1], []
    for q in range(L):
        if q == L - 1:
            T = site_matrix(kind, G, X[q], None if O is None else O[q])
            cores.append(T.reshape(T.shape[0], T.shape[1], 1))
            ranks.append(1)
            break
        r2 = X[q].shape[2]
        slabs = []
        for s in range(ls):
            t = rank * ls + s
            lo, hi = shard_range(r2, S, t)
            T = site_matrix(kind, G, X[q][:, :, lo:hi], None if O is None else O[q])   # (chi, d, w2, cnt)
            chi, d, w2, cnt = T.shape
            M = T.reshape(chi * d, w2 * cnt)
            m = M.shape[0]
            F = np.linalg.qr(M.T, mode="r") if M.shape[1] >= m else M.T
            Fp = np.zeros((mcap, mcap))
            Fp[:F.shape[0], :m] = F
            ex.send_r[s * ex.r_elems:(s + 1) * ex.r_elems] = torch.from_numpy(Fp.ravel())
            slabs.append((M, w2, cnt, lo))
        ex.allgather(0)
        recv = ex.recv_r.numpy().reshape(S, mcap, mcap)[:, :, :m]
        R = np.linalg.qr(recv.reshape(S * mcap, m), mode="r")           # the R of T^H
        U, sig, _ = np.linalg.svd(R.T)
        w2 = slabs[0][1]
        k = min(truncation_rank(sig, eps, max_rank), w2 * r2)
        delta2.append(tail_sum(sig, k))
        cores.append(U[:, :k].reshape(chi, d, k))
        ranks.append(k)
        sc = -(-r2 // S)
        for s, (M, w2, cnt, lo) in enumerate(slabs):
            Gs = np.zeros((k, w2, sc))
            Gs[:, :, :cnt] = (U[:, :k].T @ M).reshape(k, w2, cnt)
            buf = np.zeros(ex.c_elems)
            buf[:Gs.size] = Gs.ravel()
            ex.send_c[s * ex.c_elems:(s + 1) * ex.c_elems] = torch.from_numpy(buf)
        ex.allgather(1)
        recv = ex.recv_c.numpy().reshape(S, ex.c_elems)
        G = np.zeros((k, w2, r2))
        for t in range(S):
            lo, hi = shard_range(r2, S, t)
            G[:, :, lo:hi] = recv[t, :k * w2 * sc].reshape(k, w2, sc)[:, :, :hi - lo]
    return cores, ranks, delta2


def _sizes(x, S):
    mcap = max(c.shape[0] * c.shape[1] for c in x) * 2
    c_el = max(c.shape[0] * 2 * (-(-c.shape[2] // S)) for c in x) * 16
    return mcap * mcap, c_el


def _worker(rank, world, port, ls, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    kind, op, x, eps, mr = _problem()
    S = world * ls
    r_el, c_el = _sizes(x, S)
    ex = ShardExchange(world, rank, ls, r_el, c_el, "cpu", dist)
    cores, ranks, d2 = sharded_numpy(kind, op, x, eps, mr, ex, S, rank, ls)
    from oracle.tt import to_dense_vector
    out_q.put((rank, ranks, d2, to_dense_vector(cores).tolist(), ex.calls))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_partition():
    for n in (1, 3, 7, 256, 1000):
        for S in (1, 2, 3, 8):
            parts = [shard_range(n, S, t) for t in range(S)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(S - 1))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


def test_sharded_zipup_gloo_world2():
    from oracle.tt import to_dense_vector
    from oracle.zipup import zipup
    world, ls = 2, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ls, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    kind, op, x, eps, mr = _problem()
    ref = zipup(kind, op, x, eps, mr)
    yo = to_dense_vector(ref["cores"])
    L = len(x)
    for rank, ranks, d2, y, calls in res:
        assert ranks == ref["ranks"], (ranks, ref["ranks"])
        assert calls == [0, 1] * (L - 1)                 # two exchanges per split, in order
        np.testing.assert_allclose(d2, ref["delta2"], rtol=1e-9, atol=1e-12 * float(np.sum(yo ** 2)))
        assert np.linalg.norm(np.array(y) - yo) <= 1e-10 * np.linalg.norm(yo) + eps * np.linalg.norm(yo)
    assert res[0][3] == res[1][3]                           # every rank holds the same result
