"""Pins for the seeded input generators: every structured train equals its dense
definition from the paper (§4), independent of the oracle's algebra."""
import math

import numpy as np
import pytest

from paper_2602_20226_b200 import gen


def dense_vec(t):
    """Brute-force dense value: for every multi-index multiply the selected core slices
    (batched over indices, no tensor-train algebra)."""
    dims = t.dims
    N = math.prod(dims)
    c = gen.digit_factors(dims)
    n = np.arange(N)
    v = np.ones((N, 1, 1))
    for q in range(len(dims)):
        v = v @ t.cores[q][:, (n // c[q]) % dims[q], :].transpose(1, 0, 2)
    return v[:, 0, 0]


def dense_op(t):
    dims = t.dims
    N = math.prod(dims)
    c = gen.digit_factors(dims)
    i = np.repeat(np.arange(N), N)
    j = np.tile(np.arange(N), N)
    v = np.ones((N * N, 1, 1))
    for q in range(len(dims)):
        sl = t.cores[q][:, (i // c[q]) % dims[q], (j // c[q]) % dims[q], :]
        v = v @ sl.transpose(1, 0, 2)
    return v[:, 0, 0].reshape(N, N)


def test_digit_factors_and_ranks():
    assert gen.digit_factors([2, 2, 5]) == [10, 5, 1]          # SPEC.md:58 example (20 -> 2,2,5)
    assert gen.digit_factors([2, 5, 2]) == [10, 2, 1]
    assert gen.clipped_ranks([2] * 6, 4) == [1, 2, 4, 4, 4, 2, 1]
    assert gen.clipped_ranks([3] * 8 + [5] * 4, 512) == [1, 3, 9, 27, 81, 243, 512, 512, 512, 125, 25, 5, 1]


def test_exp_rank1_closed_form():
    # rank one; bases (2,3,5,2,3), domain [-1,2] endpoint-inclusive
    bases = [2, 3, 5, 2, 3]
    N = math.prod(bases)
    a, b = -1.0, 2.0
    h = (b - a) / (N - 1)
    t = gen.exp_train(bases, a, h, 1.7, 0.3)
    assert t.ranks == [1] * 6
    x = a + h * np.arange(N)
    np.testing.assert_allclose(dense_vec(t), np.exp(1.7 * (x - 0.3)), rtol=1e-14)


@pytest.mark.parametrize("fn", ["cos", "sin"])
def test_trig_rank2_closed_form(fn):
    bases = [2, 3, 5, 2, 3]
    N = math.prod(bases)
    a, b = -1.0, 2.0
    h = (b - a) / (N - 1)
    t = (gen.cos_train if fn == "cos" else gen.sin_train)(bases, a, h, 1.7, 0.3)
    assert max(t.ranks) == 2
    x = a + h * np.arange(N)
    ref = (np.cos if fn == "cos" else np.sin)(1.7 * (x - 0.3))
    np.testing.assert_allclose(dense_vec(t), ref, atol=5e-15)


def test_polynomial_rank_p_plus_1():
    bases = [2, 3, 5, 2, 3]
    N = math.prod(bases)
    a, b = -1.0, 2.0
    h = (b - a) / (N - 1)
    coeffs = [0.1, -0.4, 0.0, 1.0]
    t = gen.poly_train(bases, a, h, coeffs, 0.3)
    assert max(t.ranks) == 4
    x = a + h * np.arange(N)
    ref = sum(c * (x - 0.3) ** k for k, c in enumerate(coeffs))
    np.testing.assert_allclose(dense_vec(t), ref, atol=1e-13)


@pytest.mark.parametrize("bases", [(2, 2, 3), (2, 5, 2), (2,) * 6, (3, 3, 5), (5, 3, 3)])
def test_shift_matrices_dense(bases):
    # Q_d(i,j) = [i-j = d], R_d = Q_{N-d}^T, circular = (1,1) selection
    N = math.prod(bases)
    I = np.arange(N)[:, None]
    J = np.arange(N)[None, :]
    for d in range(N + 1):
        Q = dense_op(gen.shift_train(list(bases), d, (1.0, 0.0)))
        np.testing.assert_array_equal(Q, (I - J == d).astype(float))
        R = dense_op(gen.shift_train(list(bases), d, (0.0, 1.0)))
        np.testing.assert_array_equal(R, (J - I == N - d).astype(float))
        C = dense_op(gen.shift_train(list(bases), d, (1.0, 1.0)))
        np.testing.assert_array_equal(C, ((I - J) % N == d % N).astype(float))


def test_periodic_laplacian_rank3():
    for L in (1, 2, 3, 5):
        t = gen.periodic_laplacian_1d(L)
        assert max(t.ranks) <= 3
        N = 2 ** L
        ref = -2.0 * np.eye(N)
        for i in range(N):
            ref[i, (i + 1) % N] += 1.0
            ref[i, (i - 1) % N] += 1.0
        np.testing.assert_array_equal(dense_op(t), ref)


def test_laplacian_2d_alternating():
    Lx = 3
    t = gen.laplacian_2d_alternating(Lx)
    assert max(t.ranks) <= 6
    L1 = dense_op(gen.periodic_laplacian_1d(Lx))
    n = 2 ** Lx
    ref = np.kron(L1, np.eye(n)) + np.kron(np.eye(n), L1)   # index x*n + y
    # dense over the alternating digit layout, then permute digits x1..xn, y1..yn
    M = dense_op(t)
    L = 2 * Lx
    perm = [q for q in range(L) if q % 2 == 0] + [q for q in range(L) if q % 2 == 1]
    T = M.reshape([2] * L + [2] * L).transpose(perm + [L + q for q in perm]).reshape(n * n, n * n)
    np.testing.assert_array_equal(T, ref)


@pytest.mark.parametrize("bases", [(3, 3, 3, 5, 5), (3, 3, 3, 3, 5, 5)])
def test_stencil_rank8(bases):
    t = gen.stencil_rank8(list(bases))
    assert t.ranks[1:-1] == [8] * (len(bases) - 1)
    N = math.prod(bases)
    I = np.arange(N)[:, None]
    J = np.arange(N)[None, :]
    ref = np.zeros((N, N))
    for s, w in zip(range(-2, 3), (1.0, -4.0, 6.0, -4.0, 1.0)):
        ref += w * (I - J == s)
    np.testing.assert_array_equal(dense_op(t), ref)


def test_cfg1_state_closed_form():
    p = gen.cfg1(10)
    x = np.arange(1024) / 1024.0
    np.testing.assert_allclose(dense_vec(p.x), np.sin(2 * np.pi * x) + x * x, atol=2e-15)
    assert p.x.ranks[1:-1] == [5] * 9


def test_seeds_reproducible_and_shapes():
    a = gen.cfg5_member(3, L=12)
    b = gen.cfg5_member(3, L=12)
    c = gen.cfg5_member(4, L=12)
    for x, y in zip(a.x.cores, b.x.cores):
        np.testing.assert_array_equal(x, y)
    assert not np.array_equal(a.x.cores[5], c.x.cores[5])
    assert a.x.ranks == gen.clipped_ranks([2] * 12, 64)
    assert a.op.ranks == [1, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 1]
    # N(0, 1/R) scaling (SURVEY.md c-A14)
    big = gen.random_mps([2] * 14, 64, gen.rng_for(5, 0, 0), 1.0 / 8.0)
    allv = np.concatenate([c.ravel() for c in big.cores])
    assert abs(allv.std() - 0.125) < 0.01


def test_cfg2_normalised():
    p = gen.cfg2(Lx=4, R=8)
    assert abs(gen.env_norm(p.x) - 1.0) < 1e-13
