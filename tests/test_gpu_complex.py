"""GPU parity of the complex128 zip-up against the oracle: random
complex Hadamard / MPO / truncation zip-ups (dense comparison), and the tensorized Fourier
transform of PAPER.md:533-566 as a chain of Hadamard zip-ups -- exact on the paper's
240 x 240 example, step-by-step parity on N = 2^10, and the paper's printed N = 2^13
distances (tests/golden/qft_distances.txt, reading c-A34)."""
import math
import os

import numpy as np
import pytest

from paper_2602_20226_b200 import gen

pytestmark = pytest.mark.gpu


def _c(cores, rng):
    return [c + 1j * rng.standard_normal(c.shape) for c in cores]


def run_c(lib, subs, op, x, eps, max_rank, mpo=False):
    import torch
    xd = lib.to_device(x, dtype=np.complex128)
    od = None if op is None else lib.to_device(op, mpo=mpo, dtype=np.complex128)
    plan = lib.ZipupPlan(subs, od, xd, eps, max_rank, sigma_stride=256, sweeps=True)
    res = plan.run(od, xd)
    torch.cuda.synchronize()
    assert int(res.status.item()) == 0, int(res.status.item())
    assert res.out.cores[0].dtype == torch.complex128
    return res


def _check_dense(lib, kind, op, x, eps, max_rank, mpo=False):
    from oracle.zipup import zipup as ozip
    from oracle import tt
    subs = {"matvec": "ij,j->i", "hadamard": "i,i->i", "truncate": "i->i"}[kind]
    res = run_c(lib, subs, op, x, eps, max_rank, mpo=mpo)
    ranks = res.ranks[0].cpu().tolist()
    cores = lib.member_cores(res.out, ranks, 0)
    ref = ozip(kind, op, x, eps, max_rank)
    assert ranks == ref["ranks"]
    y, yr = tt.full_legs(cores), tt.full_legs(ref["cores"])
    assert np.linalg.norm(y - yr) <= 1e-11 * np.linalg.norm(yr)
    sig = res.sigma[0].cpu().numpy()
    for q, s in enumerate(ref["sigmas"]):
        np.testing.assert_allclose(sig[q][:len(s)], s, rtol=0, atol=1e-12 * s[0])
    np.testing.assert_allclose(res.delta2[0].cpu().numpy()[:-1], ref["delta2"], rtol=1e-8, atol=1e-24)
    assert abs(float(res.norm2[0].item()) - ref["norm"] ** 2) <= 1e-11 * ref["norm"] ** 2
    for c in cores[:-1]:                       # emitted cores are left-orthonormal (complex sense)
        M = c.reshape(-1, c.shape[-1])
        np.testing.assert_allclose(M.conj().T @ M, np.eye(M.shape[1]), atol=1e-12)


@pytest.mark.parametrize("L,R,mr,eps", [(10, 8, 6, 0.0), (9, 16, 0, 1e-6), (12, 12, 20, 1e-10)])
def test_complex_hadamard_random(lib, L, R, mr, eps):
    rng = np.random.default_rng(40 + L)
    a = _c(gen.random_mps([2] * L, R, rng, 1 / math.sqrt(R)).cores, rng)
    b = _c(gen.random_mps([2] * L, R, rng, 1 / math.sqrt(R)).cores, rng)
    _check_dense(lib, "hadamard", a, b, eps, mr)


def test_complex_matvec_mixed_radix(lib):
    rng = np.random.default_rng(41)
    dims = [2, 3, 2, 5, 2, 2]
    x = _c(gen.random_mps(dims, 9, rng).cores, rng)
    op = _c(gen.random_mpo(dims, 3, rng, 0.5).cores, rng)
    _check_dense(lib, "matvec", op, x, 1e-12, 30, mpo=True)


def test_complex_truncate(lib):
    rng = np.random.default_rng(42)
    x = _c(gen.random_mps([2] * 11, 24, rng).cores, rng)
    _check_dense(lib, "truncate", None, x, 1e-3, 0)


def _gpu_chain(lib, trains, max_rank, check_each=False):
    """Y_1 = T_1, Y_q = zip-up(T_q o Y_{q-1}) (reading c-A34), every step a qtt_zipup call;
    member_view feeds each output (zero copy) to the next call.  check_each: every step is
    compared with the oracle step on the same input by the tests/parity.py protocol (rank
    cuts at exactly-zero singular values are fragile with eps = 0, c-A9)."""
    import torch
    from parity import compare
    y = lib.to_device(trains[0], dtype=np.complex128)
    ycpu = [np.asarray(c) for c in trains[0]]
    for t in trains[1:]:
        op = lib.to_device(t, dtype=np.complex128)
        plan = lib.ZipupPlan("i,i->i", op, y, 0.0, max_rank, sigma_stride=64)
        res = plan.run(op, y)
        torch.cuda.synchronize()
        assert int(res.status.item()) == 0
        ranks = res.ranks[0].cpu().tolist()
        if check_each:
            got = lib.member_cores(res.out, ranks, 0)
            out = compare("hadamard", t, ycpu, 0.0, max_rank, got, ranks, res.sigma[0].cpu().numpy(),
                          res.delta2[0].cpu().numpy(), float(res.norm2[0].item()))
            ycpu = out["ref"]["cores"]
        y = lib.member_view(res.out, ranks, 0)
        y._keep = plan                      # the views alias the plan's output buffers
    return lib.member_cores(y, y.ranks, 0)


def test_qft_exact_240(lib):
    """The paper's 240 x 240 mixed-radix factorisation (Fig. fourier_shape): without
    truncation the chain reproduces the DFT matrix."""
    from oracle import qft
    bases = [3, 2, 2, 5, 2, 2]
    cores = _gpu_chain(lib, [t.cores for t in gen.qft_trains(bases)], 10 ** 6)
    assert qft.distance(cores, bases) <= 1e-11 * 240


@pytest.mark.parametrize("R", [2, 4, 8, 16])
def test_qft_chain_parity_2_10(lib, R):
    _gpu_chain(lib, [t.cores for t in gen.qft_trains([2] * 10)], R, check_each=True)


def test_qft_paper_distances_2_13(lib):
    """PAPER.md:566 at N = 2^13 (golden file; c-A34: distance / sqrt(N))."""
    from oracle import qft
    bases = [2] * 13
    N = 2 ** 13
    golden = os.path.join(os.path.dirname(__file__), "golden", "qft_distances.txt")
    rows = [l.split() for l in open(golden) if l.strip() and not l.startswith("#")]
    T = [t.cores for t in gen.qft_trains(bases)]
    M = qft.dft_matrix(N)
    for r, paper in rows:
        R, paper = int(r), float(paper)
        cores = _gpu_chain(lib, T, R)
        d = float(np.linalg.norm(qft.to_matrix(cores, bases) - M)) / math.sqrt(N)
        if R < 16:
            assert abs(d - paper) <= 0.06 * paper, (R, d, paper)
        else:
            assert d <= paper, (R, d, paper)


def test_complex_batch_shared_operator_and_edges(lib):
    """Batch of 3 members with one shared complex operator, a single-site train, an all-zero
    train, and inputs at 1e-140 (the Jacobi's squares stay in range)."""
    import torch
    from parity import compare
    rng = np.random.default_rng(43)
    dims = [2] * 9
    xs = [_c(gen.random_mps(dims, 10, rng).cores, rng) for _ in range(3)]
    op = _c(gen.random_mpo(dims, 3, rng, 0.5).cores, rng)
    xd = lib.to_device([np.stack([x[q] for x in xs]) for q in range(len(dims))], dtype=np.complex128)
    od = lib.to_device(op, mpo=True, dtype=np.complex128)
    plan = lib.ZipupPlan("ij,j->i", od, xd, 1e-10, 16, sigma_stride=64)
    res = plan.run(od, xd)
    torch.cuda.synchronize()
    assert int(res.status.item()) == 0
    for b in range(3):
        ranks = res.ranks[b].cpu().tolist()
        cores = lib.member_cores(res.out, ranks, b)
        compare("matvec", op, xs[b], 1e-10, 16, cores, ranks, res.sigma[b].cpu().numpy(),
                res.delta2[b].cpu().numpy(), float(res.norm2[b].item()))
    # single site
    x1 = [rng.standard_normal((1, 5, 1)) + 1j * rng.standard_normal((1, 5, 1))]
    o1 = [rng.standard_normal((1, 5, 1)) + 1j * rng.standard_normal((1, 5, 1))]
    _check_dense(lib, "hadamard", o1, x1, 0.0, 0)
    # zero input
    z = [np.zeros((1, 2, 2), complex), np.zeros((2, 2, 2), complex), np.zeros((2, 2, 1), complex)]
    r0 = run_c(lib, "i->i", None, z, 1e-8, 4)
    assert r0.ranks[0].cpu().tolist() == [1, 1, 1, 1] and float(r0.norm2[0].item()) == 0.0
    # tiny magnitudes
    a = _c(gen.random_mps([2] * 8, 6, rng).cores, rng)
    b = _c(gen.random_mps([2] * 8, 6, rng).cores, rng)
    a[0] = a[0] * 1e-140
    _check_dense(lib, "hadamard", a, b, 1e-12, 0)
