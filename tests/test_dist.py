"""Multi-process (gloo, world size 2, CPU) tests of the N>1 host path: member sharding and
the single all-reduce of the batch summary.  The per-member numbers are
produced by the oracle on small cfg5-shaped members, so the reduced totals are checked
against a single-process computation over all members."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_20226_b200 import dist as qdist
from paper_2602_20226_b200 import gen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _member_stats(b):
    from oracle.zipup import zipup
    p = gen.cfg5_member(b, L=10, R=8, W=2, max_rank=6)
    r = zipup("matvec", p.op.cores, p.x.cores, p.eps, p.max_rank)
    return r["delta2"] + [0.0], r["norm"] ** 2, r["ranks"]


def _worker(rank, world, port, M, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = qdist.member_range(rank, world, M)
    stats = [_member_stats(b) for b in range(lo, hi)]
    s = torch.tensor(qdist.local_summary([x[0] for x in stats], [x[1] for x in stats], [x[2] for x in stats]),
                     dtype=torch.float64)
    qdist.allreduce_summary(s, dist)
    t = qdist.max_over_ranks(10.0 + rank, "cpu", dist)
    out_q.put((rank, (lo, hi), s.tolist(), t))
    dist.barrier()
    dist.destroy_process_group()


def test_member_ranges_partition():
    world, M = 4, 5
    got = [qdist.member_range(r, world, M) for r in range(world)]
    assert got == [(0, 5), (5, 10), (10, 15), (15, 20)]
    for total in (7, 8, 4096):
        parts = [qdist.strong_range(r, 3, total) for r in range(3)]
        assert parts[0][0] == 0 and parts[-1][1] == total
        assert all(parts[i][1] == parts[i + 1][0] for i in range(2))
        assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


def test_allreduce_summary_gloo_world2():
    world, M = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # every rank sees the same global totals, equal to the single-process sum over all members
    stats = [_member_stats(b) for b in range(world * M)]
    ref = qdist.local_summary([x[0] for x in stats], [x[1] for x in stats], [x[2] for x in stats])
    for rank, rng, s, t in res:
        np.testing.assert_allclose(s, ref, rtol=1e-12)
        assert t == 10.0 + world - 1          # max over ranks
    assert [r[1] for r in res] == [(0, 3), (3, 6)]
    d = qdist.summary_dict(res[0][2])
    assert d["members"] == world * M
