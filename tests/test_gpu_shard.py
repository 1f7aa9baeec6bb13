"""GPU parity of the sharded zip-up (qtt_zipup_sharded) against the oracle:
one zip-up split into S column shards (R-tree of the shard factors + carry exchange).  On the
single GPU of the test box the S shards run as `local_shards` of one process (world = 1), the
exchanges either copied by the library or routed through the Python all-gather callback --
the same arithmetic and the same call sequence as S processes (the gloo world-2 CPU test
covers the multi-process exchange itself, tests/test_shard.py)."""
import math

import numpy as np
import pytest

from paper_2602_20226_b200 import gen
from parity import compare

pytestmark = pytest.mark.gpu


def run_sharded(lib, kind, op, x, eps, max_rank, local_shards, callback=None, sigma_stride=512):
    import torch
    from paper_2602_20226_b200.shard import zipup_sharded
    subs = {"matvec": "ij,j->i", "hadamard": "i,i->i", "truncate": "i->i"}[kind]
    xd = lib.to_device(x)
    od = None if op is None else lib.to_device(op, mpo=(kind == "matvec"))
    res, ex = zipup_sharded(subs, od, xd, eps, max_rank, world=1, rank=0, local_shards=local_shards,
                            sigma_stride=sigma_stride, callback=callback)
    torch.cuda.synchronize()
    assert int(res.status.item()) == 0, int(res.status.item())
    return res, ex


def check_sharded(lib, kind, op, x, eps, max_rank, local_shards, dense=True, callback=None, ref=None):
    res, ex = run_sharded(lib, kind, op, x, eps, max_rank, local_shards, callback)
    ranks = res.ranks[0].cpu().tolist()
    cores = lib.member_cores(res.out, ranks, 0)
    out = compare(kind, op, x, eps, max_rank, cores, ranks, res.sigma[0].cpu().numpy(), res.delta2[0].cpu().numpy(),
                  float(res.norm2[0].item()), dense=dense, ref=ref)
    return out, res, ex


@pytest.mark.parametrize("shards", [1, 2, 3, 5])
def test_sharded_hadamard_cfg3_shape(lib, shards):
    """configs[2] family (Hadamard of two random trains, m up to 256) split into 1-5 shards."""
    p = gen.cfg3(L=14, R=128, max_rank=128)
    check_sharded(lib, "hadamard", p.op.cores, p.x.cores, p.eps, p.max_rank, shards)


def test_sharded_matvec_and_truncate(lib):
    p = gen.cfg2(Lx=6, R=64, max_rank=128)
    check_sharded(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank, 4)
    x = gen.random_mps([3] * 7, 60, np.random.default_rng(5)).cores
    check_sharded(lib, "truncate", None, x, 1e-8, 0, 2)


def test_sharded_callback_matches_internal_exchange(lib):
    """The Python all-gather callback (the path a multi-process run takes) gives bit-identical
    results to the library's own copy, and is called twice per split in site order."""
    import torch
    p = gen.cfg3(L=12, R=64, max_rank=64)
    r1, _ = run_sharded(lib, "hadamard", p.op.cores, p.x.cores, p.eps, p.max_rank, 3, callback=False)
    r2, ex = run_sharded(lib, "hadamard", p.op.cores, p.x.cores, p.eps, p.max_rank, 3, callback=True)
    assert ex.calls == [0, 1] * (len(p.x.cores) - 1)
    assert torch.equal(r1.ranks, r2.ranks)
    for a, b in zip(r1.out.cores, r2.out.cores):
        assert torch.equal(a, b)


def test_sharded_equals_unsharded_gpu(lib):
    """Same zip-up unsharded (qtt_zipup) and in 4 shards: same ranks, results within rounding."""
    import torch
    from oracle import tt
    p = gen.cfg3(L=14, R=128, max_rank=100)
    xd, od = lib.to_device(p.x.cores), lib.to_device(p.op.cores)
    r0 = lib.ZipupPlan("i,i->i", od, xd, p.eps, p.max_rank).run(od, xd)
    torch.cuda.synchronize()
    r4, _ = run_sharded(lib, "hadamard", p.op.cores, p.x.cores, p.eps, p.max_rank, 4)
    assert r0.ranks[0].tolist() == r4.ranks[0].tolist()
    y0 = lib.member_cores(r0.out, r0.ranks[0].tolist(), 0)
    y4 = lib.member_cores(r4.out, r4.ranks[0].tolist(), 0)
    assert tt.diff_norm(y0, y4) <= 1e-10 * tt.qr_norm(y0)


@pytest.mark.slow
def test_sharded_cfg3_full_oracle_parity(lib):
    """configs[2] at full size in 2 shards (the 2-GPU split of one cfg3 zip-up) against the
    oracle (tests/golden/cache/cfg3_f64.npz or computed) by the §8(c) protocol."""
    from oracle_cache import oracle_result
    p = gen.cfg3()
    ref = oracle_result("cfg3_f64", "hadamard", p.op.cores, p.x.cores, p.eps, p.max_rank)
    out, res, ex = check_sharded(lib, "hadamard", p.op.cores, p.x.cores, p.eps, p.max_rank, 2, dense=False, ref=ref)
    print("cfg3 full, 2 shards:", {k: v for k, v in out.items() if k != "ref"})
