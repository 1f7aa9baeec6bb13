"""GPU parity of the exact operations (qtt_einsum_exact, qtt_inner, qtt_to_dense) and the
batch summary against the oracle's exact algebra (bit-for-bit up to fp64 rounding)."""
import math

import numpy as np
import pytest

from oracle import tt
from paper_2602_20226_b200 import gen

pytestmark = pytest.mark.gpu


def test_einsum_exact_matvec(lib):
    dims = [2, 3, 5, 2, 3]
    x = gen.random_mps(dims, 6, np.random.default_rng(1)).cores
    W = gen.random_mpo(dims, 3, np.random.default_rng(2)).cores
    out = lib.einsum_exact("ij,j->i", lib.to_device(W, mpo=True), lib.to_device(x))
    ref = tt.exact_matvec(W, x)
    got = lib.member_cores(out, out.ranks, 0)
    for a, b in zip(got, ref):
        np.testing.assert_allclose(a, b, rtol=1e-14, atol=1e-14)


def test_einsum_exact_hadamard(lib):
    a = gen.random_mps([2] * 9, 5, np.random.default_rng(3)).cores
    b = gen.random_mps([2] * 9, 7, np.random.default_rng(4)).cores
    out = lib.einsum_exact("i,i->i", lib.to_device(a), lib.to_device(b))
    for g, r in zip(lib.member_cores(out, out.ranks, 0), tt.exact_hadamard(a, b)):
        np.testing.assert_allclose(g, r, rtol=1e-14, atol=1e-15)


def test_inner_matches_oracle(lib):
    dims = [2] * 20
    a = gen.random_mps(dims, 32, np.random.default_rng(5)).cores
    b = gen.random_mps(dims, 17, np.random.default_rng(6)).cores
    got = float(lib.inner(lib.to_device(a), lib.to_device(b)).item())
    ref = tt.inner(a, b)
    scale = math.sqrt(tt.inner(a, a) * tt.inner(b, b))
    assert abs(got - ref) <= 1e-13 * scale
    W = gen.random_mpo([2, 3, 2], 2, np.random.default_rng(7)).cores
    g2 = float(lib.inner(lib.to_device(W, mpo=True), lib.to_device(W, mpo=True)).item())
    assert abs(g2 - tt.inner(W, W)) <= 1e-13 * abs(tt.inner(W, W))


def test_to_dense_1d_and_2d(lib):
    dims = [2, 3, 5, 2, 7]
    x = gen.random_mps(dims, 4, np.random.default_rng(8)).cores
    got = lib.to_dense(lib.to_device(x))[0].cpu().numpy()
    np.testing.assert_allclose(got, tt.to_dense_vector(x), rtol=1e-13, atol=1e-14)
    p = gen.cfg2(Lx=4, R=8)
    got = lib.to_dense(lib.to_device(p.x.cores), leg_dim=p.x.leg_dim)[0].cpu().numpy()
    np.testing.assert_allclose(got, tt.to_dense_vector(p.x.cores, p.x.leg_dim), rtol=1e-12, atol=1e-14)


def test_to_dense_guard(lib):
    x = gen.random_mps([2] * 25, 2, np.random.default_rng(9)).cores
    with pytest.raises(lib.QttError):
        lib.to_dense(lib.to_device(x))


def test_summary_fixed_order(lib):
    import torch
    probs, xs, ops = gen.cfg5_batch_arrays(range(3), L=12, R=16, W=2)
    xd, od = lib.to_device(xs), lib.to_device(ops, mpo=True)
    res = lib.ZipupPlan("ij,j->i", od, xd, 1e-10, 8).run(od, xd)
    s = lib.summary(res).cpu().numpy()
    torch.cuda.synchronize()
    d2 = res.delta2.cpu().numpy(); n2 = res.norm2.cpu().numpy(); rk = res.ranks.cpu().numpy()
    assert s[3] == 3
    assert abs(s[0] - d2.sum()) <= 1e-14 * max(d2.sum(), 1e-300)
    assert abs(s[1] - n2.sum()) <= 1e-14 * n2.sum()
    assert s[2] == rk[:, 1:-1].sum()
