"""GPU parity: qtt_zipup (through the C-ABI) vs the CPU oracle, per the comparison protocol
in tests/parity.py.  Sizes span several tiles, ragged tails, mixed radix and the
degenerate cases (L=1, L=2, zero input, max_rank=1, shared operator)."""
import math

import numpy as np
import pytest

from paper_2602_20226_b200 import gen
from parity import compare

pytestmark = pytest.mark.gpu


def run_gpu(lib, kind, op, x, eps, max_rank, mpo_op=True, flags=0, sigma_stride=256):
    import torch
    subs = {"matvec": "ij,j->i", "hadamard": "i,i->i", "truncate": "i->i"}[kind]
    xd = lib.to_device(x)
    od = None if op is None else lib.to_device(op, mpo=(kind == "matvec"))
    plan = lib.ZipupPlan(subs, od, xd, eps, max_rank, flags=flags, sigma_stride=sigma_stride)
    res = plan.run(od, xd)
    torch.cuda.synchronize()
    assert int(res.status.item()) == 0, f"device status {int(res.status.item())}"
    return res


def member(lib, res, b=0):
    ranks = res.ranks[b].cpu().tolist()
    cores = lib.member_cores(res.out, ranks, b)
    sig = res.sigma[b].cpu().numpy()
    return cores, ranks, sig, res.delta2[b].cpu().numpy(), float(res.norm2[b].item())


def check(lib, kind, op, x, eps, max_rank, dense=True, **kw):
    res = run_gpu(lib, kind, op, x, eps, max_rank, **kw)
    cores, ranks, sig, d2, n2 = member(lib, res)
    orth = not (kw.get("flags", 0) & 1)
    return compare(kind, op, x, eps, max_rank, cores, ranks, sig, d2, n2, dense=dense, orth_operator=orth)


def test_cfg1_full(lib):
    p = gen.cfg1(10)
    out = check(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank)
    # configs[0] check: dense 1024x1024 matvec / closed form (pinned in the oracle tests)
    N, h = 1024, 1.0 / 1024
    xg = np.arange(N) * h
    q = np.full(N, 2 * h * h); q[0] = h * h + (1 - h) ** 2; q[N - 1] = -1 + 2 * h * h
    closed = (2 * math.cos(2 * math.pi / N) - 2) * np.sin(2 * np.pi * xg) + q
    from oracle import tt
    res = run_gpu(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank)
    cores, ranks, *_ = member(lib, res)
    y = tt.to_dense_vector(cores)
    assert np.linalg.norm(y - closed) <= 1e-11 * np.linalg.norm(closed)


@pytest.mark.parametrize("L,R,mr,eps", [(10, 8, 4, 0.0), (12, 16, 0, 1e-3), (9, 32, 7, 1e-12), (14, 64, 48, 1e-10)])
def test_truncate_random(lib, L, R, mr, eps):
    x = gen.random_mps([2] * L, R, np.random.default_rng(L * 100 + R)).cores
    check(lib, "truncate", None, x, eps, mr, dense=(L <= 14))


@pytest.mark.parametrize("dims,R,W,mr,eps", [([2] * 12, 16, 3, 20, 1e-10), ([2, 3, 2, 5, 3, 2, 2], 9, 4, 0, 0.0),
                                             ([3] * 6 + [5] * 2, 12, 2, 30, 1e-12), ([2] * 16, 64, 4, 64, 1e-10)])
def test_matvec_random(lib, dims, R, W, mr, eps):
    x = gen.random_mps(dims, R, np.random.default_rng(len(dims) * 7 + R)).cores
    op = gen.random_mpo(dims, W, np.random.default_rng(len(dims) * 11 + W), 0.5).cores
    check(lib, "matvec", op, x, eps, mr, dense=(math.prod(dims) <= 1 << 16))


@pytest.mark.parametrize("L,R,mr,eps", [(12, 16, 32, 1e-8), (10, 8, 0, 0.0), (16, 32, 48, 1e-8)])
def test_hadamard_random(lib, L, R, mr, eps):
    a = gen.random_mps([2] * L, R, np.random.default_rng(500 + L), 1 / math.sqrt(R)).cores
    b = gen.random_mps([2] * L, R, np.random.default_rng(600 + L), 1 / math.sqrt(R)).cores
    check(lib, "hadamard", a, b, eps, mr, dense=(L <= 14))


def test_matvec_operator_not_orthonormalised(lib):
    dims = [2] * 10
    x = gen.random_mps(dims, 8, np.random.default_rng(1)).cores
    op = gen.random_mpo(dims, 3, np.random.default_rng(2)).cores
    check(lib, "matvec", op, x, 1e-8, 10, flags=1)


def test_cfg2_reduced(lib):
    p = gen.cfg2(Lx=5, R=16, max_rank=32)
    check(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank)


def test_cfg4_reduced_mixed_radix(lib):
    p = gen.cfg4(bases=(3, 3, 3, 5, 5), R=16, max_rank=24)
    check(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank)


def test_cfg3_reduced_hadamard(lib):
    p = gen.cfg3(L=14, R=32, max_rank=32)
    check(lib, "hadamard", p.op.cores, p.x.cores, p.eps, p.max_rank)


def test_cfg5_batch_members(lib):
    """configs[4] shapes (L=40, rank 64, MPO rank 4, max rank 64) on a 6-member batch;
    every member compared (QR-sweep distance: 2^40 entries cannot be densified)."""
    import torch
    members = [0, 1, 2, 511, 1000, 4095]
    probs, xs, ops = gen.cfg5_batch_arrays(members)
    xd = lib.to_device(xs)
    od = lib.to_device(ops, mpo=True)
    plan = lib.ZipupPlan("ij,j->i", od, xd, 1e-10, 64, sigma_stride=128)
    res = plan.run(od, xd)
    torch.cuda.synchronize()
    assert int(res.status.item()) == 0
    for i, p in enumerate(probs):
        cores, ranks, sig, d2, n2 = member(lib, res, i)
        compare("matvec", p.op.cores, p.x.cores, p.eps, p.max_rank, cores, ranks, sig, d2, n2, dense=False)


def test_edge_single_site(lib):
    x = [np.random.default_rng(3).standard_normal((1, 5, 1))]
    op = [np.random.default_rng(4).standard_normal((1, 5, 5, 1))]
    check(lib, "matvec", op, x, 0.0, 0)


def test_edge_two_sites_and_rank1(lib):
    x = gen.random_mps([3, 2], 3, np.random.default_rng(5)).cores
    check(lib, "truncate", None, x, 0.0, 1)
    x = gen.random_mps([2] * 9, 8, np.random.default_rng(6)).cores
    check(lib, "truncate", None, x, 0.0, 1)


def test_edge_zero_input(lib):
    x = [np.zeros((1, 2, 2)), np.zeros((2, 2, 2)), np.zeros((2, 2, 1))]
    res = run_gpu(lib, "truncate", None, x, 1e-8, 4)
    cores, ranks, sig, d2, n2 = member(lib, res)
    assert ranks == [1, 1, 1, 1] and n2 == 0.0 and np.all(d2 == 0.0)


def test_shared_operator_batch(lib):
    import torch
    dims = [2] * 12
    xs = [gen.random_mps(dims, 16, np.random.default_rng(70 + b)).cores for b in range(3)]
    op = gen.random_mpo(dims, 3, np.random.default_rng(80)).cores
    xd = lib.to_device([np.stack([x[q] for x in xs]) for q in range(12)])
    od = lib.to_device(op, mpo=True)       # batch 1: shared by every member
    plan = lib.ZipupPlan("ij,j->i", od, xd, 1e-10, 24, sigma_stride=64)
    res = plan.run(od, xd)
    torch.cuda.synchronize()
    for b in range(3):
        cores, ranks, sig, d2, n2 = member(lib, res, b)
        compare("matvec", op, xs[b], 1e-10, 24, cores, ranks, sig, d2, n2)


def test_nonfinite_input_flagged(lib):
    x = gen.random_mps([2] * 8, 4, np.random.default_rng(9)).cores
    x[3] = x[3].copy(); x[3][0, 0, 0] = np.nan
    import torch
    xd = lib.to_device(x)
    res = lib.ZipupPlan("i->i", None, xd, 1e-8, 4).run(None, xd)
    torch.cuda.synchronize()
    assert int(res.status.item()) & 1


def test_round_after_zipup_reaches_minimal_ranks(lib):
    """f1: qtt_round on the cfg1 zip-up output == oracle round_train, and the ranks equal the
    numerical ranks of the dense result's unfoldings."""
    import torch
    from oracle import tt
    from oracle.zipup import zipup as ozip
    p = gen.cfg1(10)
    res = run_gpu(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank)
    rr = lib.round_train(res.out, res.ranks, 1e-12, 0)
    torch.cuda.synchronize()
    assert int(rr.status.item()) == 0
    ranks = rr.ranks[0].cpu().tolist()
    y = lib.member_cores(rr.out, ranks, 0)
    ref_zip = ozip("matvec", p.op.cores, p.x.cores, p.eps, p.max_rank)
    ref = tt.round_train(ref_zip["cores"], 1e-12, 0)
    assert ranks == tt.ranks_of(ref)
    yd = tt.to_dense_vector(ref_zip["cores"])
    dense_ranks = [tt.truncation_rank(np.linalg.svd(yd.reshape(2 ** k, -1), compute_uv=False), 1e-12, 0)
                   for k in range(1, 10)]
    assert ranks[1:-1] == dense_ranks
    yv, rv = tt.to_dense_vector(y), tt.to_dense_vector(ref)
    assert np.linalg.norm(yv - rv) <= 1e-10 * np.linalg.norm(rv)


def test_round_redundant_and_max_rank(lib):
    """Rounding a redundant representation (x + x, formal rank 2r) to max_rank: equals the
    oracle's rounding of the same train."""
    import torch
    from oracle import tt
    x = gen.random_mps([2, 3, 2, 2, 3, 2], 4, np.random.default_rng(21)).cores
    xx = tt.add(x, x)
    xd = lib.to_device(xx)
    for mr, eps in ((0, 1e-12), (3, 0.0)):
        rr = lib.round_train(xd, None, eps, mr)
        torch.cuda.synchronize()
        ranks = rr.ranks[0].cpu().tolist()
        ref = tt.round_train(xx, eps, mr)
        assert ranks == tt.ranks_of(ref)
        yv, rv = tt.to_dense_vector(lib.member_cores(rr.out, ranks, 0)), tt.to_dense_vector(ref)
        assert np.linalg.norm(yv - rv) <= 1e-10 * np.linalg.norm(rv)


def test_host_pipeline_batches(lib):
    """qtt.HostPipeline: three different host batches streamed through two buffer sets; each
    batch's host-side results (copied back by the pipeline) match the oracle."""
    import torch
    dims = [2] * 10
    batches = []
    for k in range(3):
        xs = [gen.random_mps(dims, 12, np.random.default_rng(900 + 10 * k + b)).cores for b in range(2)]
        ops = [gen.random_mpo(dims, 3, np.random.default_rng(950 + 10 * k + b), 0.5).cores for b in range(2)]
        batches.append((xs, ops))
    stack = lambda ts: [np.stack([t[q] for t in ts]) for q in range(len(dims))]
    xd = lib.to_device(stack(batches[0][0]))
    od = lib.to_device(stack(batches[0][1]), mpo=True)
    pipe = lib.HostPipeline("ij,j->i", od, xd, 1e-10, 16, depth=2)
    plan0 = pipe.sets[0][2]
    hosts = []
    pipe.begin()
    for xs, ops in batches:
        hx = [torch.from_numpy(c).pin_memory() for c in stack(xs)]
        ho = [torch.from_numpy(c).pin_memory() for c in stack(ops)]
        hout = [torch.empty(c.shape, dtype=c.dtype).pin_memory() for c in plan0.out.cores]
        hr = torch.empty(tuple(plan0.ranks.shape), dtype=torch.int32).pin_memory()
        hd = torch.empty(tuple(plan0.delta2.shape), dtype=torch.float64).pin_memory()
        hn = torch.empty(tuple(plan0.norm2.shape), dtype=torch.float64).pin_memory()
        pipe.step(hx, ho, hout, hr, hd, hn)
        hosts.append((hx, ho, hout, hr, hd, hn))
    pipe.finish()
    torch.cuda.synchronize()
    from oracle.zipup import zipup as ozip
    from oracle import tt
    for (xs, ops), (_, _, hout, hr, hd, hn) in zip(batches, hosts):
        for b in range(2):
            ranks = hr[b].tolist()
            cores = [hout[q][b].reshape(-1)[:ranks[q] * 2 * ranks[q + 1]].numpy().reshape(ranks[q], 2, ranks[q + 1])
                     for q in range(len(dims))]
            ref = ozip("matvec", ops[b], xs[b], 1e-10, 16)
            assert ranks == ref["ranks"]
            y, yr = tt.to_dense_vector(cores), tt.to_dense_vector(ref["cores"])
            assert np.linalg.norm(y - yr) <= 1e-11 * np.linalg.norm(yr)
            assert abs(float(hn[b]) - ref["norm"] ** 2) <= 1e-11 * ref["norm"] ** 2


@pytest.mark.parametrize("scale", [1e-140, 1e140])
def test_extreme_magnitudes(lib, scale):
    """Inputs scaled to 1e-140 / 1e+140 (norm^2 near the fp64 range ends): the Jacobi's
    squared tests (g^2 vs a b) would under/overflow without its power-of-two prescale."""
    dims = [2] * 12
    x = gen.random_mps(dims, 16, np.random.default_rng(31)).cores
    x[0] = x[0] * scale
    op = gen.random_mpo(dims, 3, np.random.default_rng(32), 0.5).cores
    check(lib, "matvec", op, x, 1e-10, 24)


@pytest.mark.parametrize("R", [64, 65])
def test_small_large_path_boundary(lib, R):
    """m = chi d = 128 runs on the small-member path, 130 on the large one: both agree with the
    oracle at the boundary (SURVEY.md §8(a) a3/a4 size split)."""
    x = gen.random_mps([2] * 14, R, np.random.default_rng(100 + R)).cores      # bonds up to R
    assert max(c.shape[0] for c in x) == R
    op = gen.random_mpo([2] * 14, 2, np.random.default_rng(200 + R), 0.5).cores
    check(lib, "truncate", None, x, 1e-10, 0, dense=True)                       # m = 2 R
    check(lib, "matvec", op, x, 1e-10, 64, dense=True)


def test_maximum_sites_and_refusal(lib):
    """L = 64 sites (kMaxSites) works; L = 65 is refused with QTT_EUNSUPPORTED, not run."""
    x = gen.random_mps([2] * 64, 6, np.random.default_rng(7)).cores
    check(lib, "truncate", None, x, 1e-8, 5, dense=False)
    x65 = gen.random_mps([2] * 65, 2, np.random.default_rng(8)).cores
    xd = lib.to_device(x65)
    with pytest.raises(lib.QttError) as e:
        lib.ZipupPlan("i->i", None, xd, 1e-8, 4)
    assert e.value.status == 8


@pytest.mark.parametrize("kind", ["truncate", "matvec"])
def test_a1_blocked_rank_deficient(lib, kind):
    """a1's blocked Householder path (qr_std.cuh: M^T with 65..128 rows, 17..64 columns) on
    rank-deficient cores: a core whose M^T has duplicated columns (zero pivots in R, reflectors
    with tau = 0 further on), one with zero rows of M (zero columns of M^T), one tiny core.  The
    result must match the oracle like any other input (c-A3)."""
    dims = [2] * 12
    x = gen.random_mps(dims, 48, np.random.default_rng(77)).cores
    assert any(c.shape[0] >= 17 and c.shape[1] * c.shape[2] > 64 for c in x)
    x[5] = x[5].copy(); x[5][: x[5].shape[0] // 2] = x[5][x[5].shape[0] // 2: 2 * (x[5].shape[0] // 2)]
    x[7] = x[7].copy(); x[7][::3] = 0.0
    x[8] = x[8] * 1e-9
    op = gen.random_mpo(dims, 2, np.random.default_rng(78), 0.5).cores
    if kind == "truncate":
        check(lib, "truncate", None, x, 1e-10, 0, dense=True)
    else:
        check(lib, "matvec", op, x, 1e-10, 40, dense=True)
