"""Pins for oracle/tt.py against dense brute force, closed forms and identities."""
import math

import numpy as np
import pytest

from oracle import tt
from paper_2602_20226_b200 import gen

from test_gen import dense_op, dense_vec


def rnd(dims, R, seed, std=1.0):
    return gen.random_mps(dims, R, np.random.default_rng(seed), std).cores


def test_full_legs_matches_brute_force():
    dims = [2, 3, 2, 5]
    c = rnd(dims, 4, 1)
    v = tt.to_dense_vector(c)
    np.testing.assert_allclose(v, dense_vec(gen.Train(c)), rtol=1e-13, atol=1e-14)
    # evaluate at every multi-index equals dense
    f = gen.digit_factors(dims)
    n = np.arange(math.prod(dims))
    digs = np.stack([(n // f[q]) % dims[q] for q in range(4)], axis=1)
    np.testing.assert_allclose(tt.evaluate(c, digs), v, rtol=1e-13, atol=1e-14)


def test_dense_matrix_matches_brute_force():
    t = gen.random_mpo([2, 3, 2], 3, np.random.default_rng(2))
    np.testing.assert_allclose(tt.to_dense_matrix(t.cores), dense_op(t), rtol=1e-13, atol=1e-14)


def test_inner_and_cauchy_schwarz():
    a = rnd([2] * 8, 4, 3)
    b = rnd([2] * 8, 5, 4)
    va, vb = tt.to_dense_vector(a), tt.to_dense_vector(b)
    assert abs(tt.inner(a, b) - va @ vb) <= 1e-12 * np.linalg.norm(va) * np.linalg.norm(vb)
    assert abs(tt.inner(a, a) - va @ va) <= 1e-12 * (va @ va)
    assert abs(tt.inner(a, b)) <= math.sqrt(tt.inner(a, a) * tt.inner(b, b)) * (1 + 1e-12)
    ones = [np.ones((1, 2, 1))] * 8
    assert abs(tt.inner(ones, a) - va.sum()) <= 1e-12 * np.abs(va).sum()


def test_add_ranks_and_values():
    a, b = rnd([2] * 6, 2, 5), rnd([2] * 6, 3, 6)
    s = tt.add(a, b)
    assert tt.ranks_of(s)[1:-1] == [4, 5, 5, 5, 4]  # min(2,..)+min(3,..)
    np.testing.assert_allclose(tt.to_dense_vector(s), tt.to_dense_vector(a) + tt.to_dense_vector(b),
                               rtol=1e-13, atol=1e-13)


def test_exact_matvec_dense_and_rank_product():
    x = rnd([2, 3, 2, 2], 3, 7)
    W = gen.random_mpo([2, 3, 2, 2], 2, np.random.default_rng(8))
    y = tt.exact_matvec(W.cores, x)
    np.testing.assert_allclose(tt.to_dense_vector(y), dense_op(W) @ tt.to_dense_vector(x),
                               rtol=1e-12, atol=1e-12)
    assert tt.ranks_of(y) == [a * b for a, b in zip(W.ranks, tt.ranks_of(x))]


def test_exact_matvec_shift_example():
    # shift(dim 8, d=1, non-circular) @ ones -> (0,1,1,1,1,1,1,1)
    Q = gen.shift_train([2, 2, 2], 1)
    ones = [np.ones((1, 2, 1))] * 3
    np.testing.assert_array_equal(tt.to_dense_vector(tt.exact_matvec(Q.cores, ones)),
                                  [0, 1, 1, 1, 1, 1, 1, 1])


def test_exact_matmat_shift_algebra():
    # Q_1 Q_2 = Q_3 on dim 12
    b = [2, 2, 3]
    P = tt.exact_matmat(gen.shift_train(b, 1).cores, gen.shift_train(b, 2).cores)
    np.testing.assert_array_equal(tt.to_dense_matrix(P), dense_op(gen.shift_train(b, 3)))


def test_exact_hadamard():
    a, b = rnd([2] * 7, 2, 9), rnd([2] * 7, 3, 10)
    h = tt.exact_hadamard(a, b)
    assert max(tt.ranks_of(h)) == 6
    np.testing.assert_allclose(tt.to_dense_vector(h), tt.to_dense_vector(a) * tt.to_dense_vector(b),
                               rtol=1e-12, atol=1e-13)


def test_right_orthonormalize_keeps_value():
    x = rnd([2, 3, 2, 2, 3], 6, 11)
    y = tt.right_orthonormalize(x)
    np.testing.assert_allclose(tt.to_dense_vector(y), tt.to_dense_vector(x), rtol=1e-12, atol=1e-13)
    for c in y[1:]:
        assert tt.is_right_orthonormal(c)
    # norm lives in the first core
    assert abs(np.linalg.norm(y[0]) - np.linalg.norm(tt.to_dense_vector(x))) < 1e-12 * np.linalg.norm(y[0])
    W = gen.random_mpo([2, 2, 2], 3, np.random.default_rng(12)).cores
    Wo = tt.right_orthonormalize(W)
    np.testing.assert_allclose(tt.to_dense_matrix(Wo), tt.to_dense_matrix(W), rtol=1e-12, atol=1e-12)
    for c in Wo[1:]:
        assert tt.is_right_orthonormal(c)


def test_qr_norm_resolves_tiny_differences():
    # QR-sweep distance resolves 1e-13 relative differences
    x = rnd([2] * 10, 8, 13)
    nx = np.linalg.norm(tt.to_dense_vector(x))
    assert abs(tt.qr_norm(x) - nx) < 1e-13 * nx
    for rho in (1e-6, 1e-11, 1e-13):
        y = [c.copy() for c in x]
        y[4] = y[4] + rho * np.linalg.norm(y[4]) * np.random.default_rng(14).standard_normal(y[4].shape)
        dense = np.linalg.norm(tt.to_dense_vector(x) - tt.to_dense_vector(y)) / nx
        got = tt.diff_norm(x, y) / nx
        assert abs(got - dense) <= 0.05 * dense + 2e-15


def test_truncation_rule_examples():
    # SPEC.md:302-303
    assert tt.truncation_rank(np.ones(4), 0.0, 0) == 4
    assert tt.truncation_rank(np.array([3.0, 0, 0, 0]), 0.5, 0) == 1
    assert tt.truncation_rank(np.zeros(5), 0.1, 0) == 1
    s = np.array([1.0, 0.1, 0.01, 0.001])
    # tail after k=2: sqrt(1e-4 + 1e-6) = 0.01005 -> needs eps >= 0.01005/||s||
    tot = math.sqrt((s * s).sum())
    assert tt.truncation_rank(s, 0.0101 / tot, 0) == 2
    assert tt.truncation_rank(s, 0.0100 / tot, 0) == 3
    assert tt.truncation_rank(s, 0.0101 / tot, 1) == 1
    assert tt.truncation_rank(s, 0.0, 0) == 4


def test_tt_svd_error_identity():
    v = np.random.default_rng(15).standard_normal(2 ** 10)
    cores, d2 = tt.tt_svd(v, [2] * 10, 0.0, 0)
    np.testing.assert_allclose(tt.to_dense_vector(cores), v, rtol=1e-12, atol=1e-12)
    cores, d2 = tt.tt_svd(v, [2] * 10, 0.0, 4)
    err2 = np.sum((tt.to_dense_vector(cores) - v) ** 2)
    assert abs(err2 - sum(d2)) <= 1e-10 * err2       # TT-SVD orthogonality: equality


def test_round_gives_minimal_ranks_of_cfg1_state():
    # numerical ranks of sin(2 pi x)+x^2 unfoldings are [2,4,5,5,5,5,5,4,2]
    p = gen.cfg1(10)
    v = tt.to_dense_vector(p.x.cores)
    dense_ranks = []
    for q in range(1, 10):
        s = np.linalg.svd(v.reshape(2 ** q, -1), compute_uv=False)
        dense_ranks.append(tt.truncation_rank(s, 1e-12, 0))
    r = tt.round_train(p.x.cores, 1e-12, 0)
    assert tt.ranks_of(r)[1:-1] == dense_ranks == [2, 4, 5, 5, 5, 5, 5, 4, 2]
    assert np.max(np.abs(tt.to_dense_vector(r) - v)) < 1e-12


def test_hadamard_closed_forms_after_rounding():
    # exp*exp is exp (rank 1); cos*cos = 1/2 + 1/2 cos(2t) (rank 3), SURVEY.md A8
    b = [2] * 10
    h = 1.0 / 1024
    e = tt.exact_hadamard(gen.exp_train(b, 0, h, 0.7, 0).cores, gen.exp_train(b, 0, h, -1.3, 0).cores)
    assert max(tt.ranks_of(tt.round_train(e, 1e-12, 0))) == 1
    c = gen.cos_train(b, 0, h, 3.0, 0).cores
    cc = tt.round_train(tt.exact_hadamard(c, c), 1e-12, 0)
    assert tt.ranks_of(cc)[1:-1] == [min(3, 2 ** q, 2 ** (10 - q)) for q in range(1, 10)]


# ---------------------------------------------------------------- multi-dimension digit order
# to_tensor is row-major over the original dimensions (dimension 0 slowest),
# the digits of each dimension most significant first.  These pins build trains whose dense
# value is known in closed form per dimension, so a swapped dimension order, a reversed digit
# order or a transposed operator fails them.

def _kron_digits(factors):
    """Dense vector of prod_q f_q(digit_q), digits big-endian: kron(f_0, f_1, ...)."""
    v = np.ones(1)
    for f in factors:
        v = np.kron(v, f)
    return v


def _rank1(vecs):
    return [np.asarray(f, dtype=float).reshape(1, -1, 1) for f in vecs]


def test_dim_order_separable_interleaved_2d():
    """f(x) g(y) on the alternating layout x1,y1,x2,y2,... (configs[1], c-A19) equals
    np.outer(f, g).ravel(); f and g are general rank-2/3 trains, the other dimension's bond
    passing through each core (Kronecker bonds)."""
    rng = np.random.default_rng(11)
    Lx = 3
    F = gen.random_mps([2] * Lx, 2, rng).cores
    G = gen.random_mps([2] * Lx, 3, rng).cores
    f, g = tt.to_dense_vector(F), tt.to_dense_vector(G)
    cores, leg_dim = [], []
    for q in range(Lx):
        # x-site: C[(a,b), i, (a',b)] = F_q[a,i,a'] with g's bond b (left bond of G_q) carried
        rb = G[q].shape[0]
        cores.append(np.einsum("aic,bd->abicd", F[q], np.eye(rb)).reshape(
            F[q].shape[0] * rb, 2, F[q].shape[2] * rb))
        leg_dim.append(0)
        ra = F[q].shape[2]
        cores.append(np.einsum("ac,bid->abicd", np.eye(ra), G[q]).reshape(
            ra * G[q].shape[0], 2, ra * G[q].shape[2]))
        leg_dim.append(1)
    got = tt.to_dense_vector(cores, leg_dim)
    np.testing.assert_allclose(got, np.outer(f, g).ravel(), rtol=1e-13, atol=1e-14)
    # the swapped order is a different vector (the pin discriminates)
    assert np.abs(got - np.outer(g, f).ravel()).max() > 1e-3


def test_dim_order_three_dims_mixed_radix():
    """Three dimensions with mixed digit sizes, sites in the order z0, x0, y0, x1, z1
    (leg_dim = [2, 0, 1, 0, 2]): dense = f(x) (x) g(y) (x) h(z), row-major x slowest."""
    rng = np.random.default_rng(12)
    fx = [rng.standard_normal(3), rng.standard_normal(2)]
    gy = [rng.standard_normal(5)]
    hz = [rng.standard_normal(2), rng.standard_normal(3)]
    sites = [hz[0], fx[0], gy[0], fx[1], hz[1]]
    leg_dim = [2, 0, 1, 0, 2]
    got = tt.to_dense_vector(_rank1(sites), leg_dim)
    want = np.kron(np.kron(_kron_digits(fx), _kron_digits(gy)), _kron_digits(hz))
    np.testing.assert_allclose(got, want, rtol=1e-14, atol=0)
    # default order (site order) is the plain kron of the sites
    np.testing.assert_allclose(tt.to_dense_vector(_rank1(sites)), _kron_digits(sites), rtol=1e-14)


def test_dim_order_operator_kron():
    """A separable MPO A(x) (x) B(y) on the alternating layout densifies to np.kron(A, B)
    (rows: out indices, row-major x slowest; columns likewise)."""
    rng = np.random.default_rng(13)
    Ax = [rng.standard_normal((2, 2)) for _ in range(2)]
    By = [rng.standard_normal((3, 3)) for _ in range(2)]
    cores = [Ax[0], By[0], Ax[1], By[1]]
    mpo = [c.reshape(1, *c.shape, 1) for c in cores]
    A = np.kron(Ax[0], Ax[1])
    B = np.kron(By[0], By[1])
    np.testing.assert_allclose(tt.to_dense_matrix(mpo, [0, 1, 0, 1]), np.kron(A, B), rtol=1e-14)
    np.testing.assert_allclose(tt.to_dense_matrix(mpo), np.kron(np.kron(Ax[0], By[0]),
                                                                np.kron(Ax[1], By[1])), rtol=1e-14)


# ---------------------------------------------------------------- complex trains
# The oracle takes complex128 since f2; addition and the
# inner product (conjugate-linear in the first argument) must
# keep imaginary parts.

def _crnd(dims, R, seed):
    rng = np.random.default_rng(seed)
    re = gen.random_mps(dims, R, rng).cores
    im = gen.random_mps(dims, R, rng).cores
    return [a + 1j * b for a, b in zip(re, im)]


def test_complex_add_inner_diff_norm():
    a, b = _crnd([2, 3, 2, 2, 3], 3, 21), _crnd([2, 3, 2, 2, 3], 2, 22)
    va, vb = tt.to_dense_vector(a), tt.to_dense_vector(b)
    s = tt.add(a, b)
    assert all(np.iscomplexobj(c) for c in s)
    np.testing.assert_allclose(tt.to_dense_vector(s), va + vb, rtol=1e-13, atol=1e-13)
    ip = tt.inner(a, b)
    assert isinstance(ip, complex)
    assert abs(ip - np.vdot(va, vb)) <= 1e-12 * np.linalg.norm(va) * np.linalg.norm(vb)
    # conjugate-linear in the first argument: <i a, b> = -i <a, b>
    ia = tt.scale(a, 1j)
    assert abs(tt.inner(ia, b) - (-1j) * ip) <= 1e-12 * abs(ip)
    assert abs(tt.inner(a, a).imag) <= 1e-12 * abs(tt.inner(a, a))
    dn = tt.diff_norm(a, b)
    assert abs(dn - np.linalg.norm(va - vb)) <= 1e-12 * np.linalg.norm(va - vb)
    # a train differing from a only by an imaginary perturbation is at that distance
    c = [x.copy() for x in a]
    c[2] = c[2] + 1e-3j * np.ones_like(c[2])
    vc = tt.to_dense_vector(c)
    assert abs(tt.diff_norm(a, c) - np.linalg.norm(va - vc)) <= 1e-10 * np.linalg.norm(va - vc)
