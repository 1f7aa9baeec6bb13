"""GPU parity of qtt_variational (f3) against oracle/variational.py started
from the same seed (the GPU zip-up result): the |C_q|^2 sequence of every update, the final
ranks and the final train (dense), plus the never-increasing distance; MPO, Hadamard,
truncation, mixed radix and a batch with a shared operator; a cfg5-shape member."""
import numpy as np
import pytest

from paper_2602_20226_b200 import gen

pytestmark = pytest.mark.gpu


def _run(lib, kind, op, x, eps, max_rank, sweeps, mpo=False, vkw=None):
    import torch
    subs = {"matvec": "ij,j->i", "hadamard": "i,i->i", "truncate": "i->i"}[kind]
    xd = lib.to_device(x)
    od = None if op is None else lib.to_device(op, mpo=mpo)
    z = lib.ZipupPlan(subs, od, xd, eps, max_rank).run(od, xd)
    v = lib.variational(subs, od, xd, z, sweeps, **(vkw or {}))
    torch.cuda.synchronize()
    assert int(z.status.item()) == 0 and int(v.status.item()) == 0
    return z, v


def _check(lib, kind, op, xs, z, v, sweeps, b=0, dense=True, ncores=1, eps=0.0, max_rank=0):
    from oracle import tt
    from oracle.variational import variational as ovar
    seed = lib.member_cores(z.out, z.ranks[b].cpu().tolist(), b)
    ref = ovar(kind, op, xs, seed, sweeps, ncores=ncores, eps=eps, max_rank=max_rank)
    got_n = v.center_norm2[b].cpu().numpy()[:len(ref["center_norm2"])]
    ref_n = np.array(ref["center_norm2"])
    scale = ref_n.max()
    np.testing.assert_allclose(got_n, ref_n, rtol=0, atol=1e-10 * scale)
    assert all(got_n[i + 1] >= got_n[i] - 1e-12 * scale for i in range(len(got_n) - 1))
    ranks = v.ranks[b].cpu().tolist()
    assert ranks == [1] + [c.shape[-1] for c in ref["cores"]]
    cores = lib.member_cores(v.out, ranks, b)
    if dense:
        y, yr = tt.full_legs(cores), tt.full_legs(ref["cores"])
        assert np.linalg.norm(y - yr) <= 1e-10 * np.linalg.norm(yr)
    else:
        assert tt.diff_norm(cores, ref["cores"]) <= 1e-10 * tt.qr_norm(ref["cores"])


@pytest.mark.parametrize("kind", ["matvec", "hadamard", "truncate"])
def test_variational_random(lib, kind):
    rng = np.random.default_rng(70)
    dims = [2, 3, 2, 2, 5, 2, 2, 3]
    x = gen.random_mps(dims, 9, rng).cores
    op = {"matvec": gen.random_mpo(dims, 3, rng, 0.5).cores, "hadamard": gen.random_mps(dims, 3, rng).cores,
          "truncate": None}[kind]
    z, v = _run(lib, kind, op, x, 0.1, 6, 3, mpo=(kind == "matvec"))
    _check(lib, kind, op, x, z, v, 3)


def test_variational_batch_shared_operator(lib):
    import torch
    dims = [2] * 10
    xs = [gen.random_mps(dims, 10, np.random.default_rng(80 + b)).cores for b in range(3)]
    op = gen.random_mpo(dims, 3, np.random.default_rng(90), 0.5).cores
    xd = lib.to_device([np.stack([x[q] for x in xs]) for q in range(len(dims))])
    od = lib.to_device(op, mpo=True)
    z = lib.ZipupPlan("ij,j->i", od, xd, 0.05, 8).run(od, xd)
    v = lib.variational("ij,j->i", od, xd, z, 2)
    torch.cuda.synchronize()
    for b in range(3):
        _check(lib, "matvec", op, xs[b], z, v, 2, b=b)


def test_variational_cfg5_member(lib):
    """configs[4] shapes (L = 40, rank 64, MPO rank 4) seeded with a max-rank-16 zip-up."""
    probs, xs, ops = gen.cfg5_batch_arrays([3])
    p = probs[0]
    z, v = _run(lib, "matvec", p.op.cores, p.x.cores, 1e-10, 16, 1, mpo=True)
    _check(lib, "matvec", p.op.cores, p.x.cores, z, v, 1, dense=False)


# ------------------------------------------------------------ two-site super-cores (ncores = 2)
# PAPER.md:300 (multi-core strategies, rank control), PAPER.md:794 (ncores=2, cutoff=0.0,
# max_rank=8); reading c-A37.

@pytest.mark.parametrize("kind", ["matvec", "hadamard", "truncate"])
def test_variational_two_site_random(lib, kind):
    rng = np.random.default_rng(170)
    dims = [2, 3, 2, 2, 5, 2, 2, 3]
    x = gen.random_mps(dims, 9, rng).cores
    op = {"matvec": gen.random_mpo(dims, 3, rng, 0.5).cores, "hadamard": gen.random_mps(dims, 3, rng).cores,
          "truncate": None}[kind]
    z, v = _run(lib, kind, op, x, 0.2, 4, 2, mpo=(kind == "matvec"), vkw=dict(ncores=2, eps=0.0, max_rank=8))
    _check(lib, kind, op, x, z, v, 2, ncores=2, eps=0.0, max_rank=8)
    assert max(v.ranks[0].cpu().tolist()) > 4          # the ranks adapted beyond the seed's


def test_variational_two_site_cutoff_and_paper_call(lib):
    """The paper's call (max_rank=8, cutoff=0.0, ncores=2, nsweeps=2) and a cutoff
    that decides ranks below max_rank."""
    rng = np.random.default_rng(171)
    dims = [2] * 10
    x = gen.random_mps(dims, 6, rng).cores
    op = gen.random_mpo(dims, 2, rng, 0.5).cores
    z, v = _run(lib, "matvec", op, x, 0.3, 2, 2, mpo=True, vkw=dict(ncores=2, eps=0.0, max_rank=8))
    _check(lib, "matvec", op, x, z, v, 2, ncores=2, eps=0.0, max_rank=8)
    z, v = _run(lib, "matvec", op, x, 0.3, 2, 2, mpo=True, vkw=dict(ncores=2, eps=1e-3, max_rank=0))
    _check(lib, "matvec", op, x, z, v, 2, ncores=2, eps=1e-3, max_rank=0)


def test_variational_two_site_cfg5_member(lib):
    """configs[4] shapes seeded with a max-rank-8 zip-up, two-site sweep to max rank 16."""
    probs, xs, ops = gen.cfg5_batch_arrays([4])
    p = probs[0]
    z, v = _run(lib, "matvec", p.op.cores, p.x.cores, 1e-10, 8, 1, mpo=True, vkw=dict(ncores=2, eps=0.0, max_rank=16))
    _check(lib, "matvec", p.op.cores, p.x.cores, z, v, 1, dense=False, ncores=2, eps=0.0, max_rank=16)
