"""Pins for oracle/zipup.py (§3.2): limits, closed forms, dense TT-SVD identities
and the error bounds of SURVEY.md c-A11."""
import math

import numpy as np
import pytest

from oracle import tt
from oracle.zipup import zipup
from paper_2602_20226_b200 import gen

from test_gen import dense_op


def rnd(dims, R, seed, std=1.0):
    return gen.random_mps(dims, R, np.random.default_rng(seed), std).cores


def test_eps0_equals_exact_matvec():
    # Exact is the cutoff-0, unbounded-rank limit of Decomposition
    dims = [2, 3, 2, 2, 3, 2]
    x = rnd(dims, 5, 1)
    W = gen.random_mpo(dims, 3, np.random.default_rng(2))
    r = zipup("matvec", W.cores, x, 0.0, 0)
    ref = dense_op(W) @ tt.to_dense_vector(x)
    y = tt.to_dense_vector(r["cores"])
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)
    assert abs(r["norm"] - np.linalg.norm(ref)) <= 1e-12 * np.linalg.norm(ref)
    for c in r["cores"][:-1]:
        assert tt.is_left_orthonormal(c)


def test_eps0_equals_exact_hadamard():
    a, b = rnd([2] * 9, 6, 3), rnd([2] * 9, 5, 4)
    r = zipup("hadamard", a, b, 0.0, 0)
    ref = tt.to_dense_vector(a) * tt.to_dense_vector(b)
    assert np.linalg.norm(tt.to_dense_vector(r["cores"]) - ref) <= 1e-12 * np.linalg.norm(ref)


def test_cfg1_dense_and_closed_form():
    # configs[0]: checked against a dense 1024x1024 matvec; closed form SURVEY.md §8(c)
    p = gen.cfg1(10)
    r = zipup("matvec", p.op.cores, p.x.cores, p.eps, p.max_rank)
    y = tt.to_dense_vector(r["cores"])
    N, h = 1024, 1.0 / 1024
    xg = np.arange(N) * h
    M = dense_op(p.op)
    ref = M @ (np.sin(2 * np.pi * xg) + xg * xg)
    q = np.full(N, 2 * h * h)
    q[0] = h * h + (1 - h) ** 2
    q[N - 1] = -1 + 2 * h * h
    closed = (2 * math.cos(2 * math.pi / N) - 2) * np.sin(2 * np.pi * xg) + q
    np.testing.assert_allclose(ref, closed, atol=2e-15)
    assert np.linalg.norm(y - closed) <= 1e-11 * np.linalg.norm(closed)
    assert max(r["ranks"]) <= 16
    # rounding the zip-up output reaches the dense numerical ranks of y (A8 / f1)
    dense_ranks = [tt.truncation_rank(np.linalg.svd(closed.reshape(2 ** k, -1), compute_uv=False), 1e-12, 0)
                   for k in range(1, 10)]
    rr = tt.round_train(r["cores"], 1e-12, 0)
    assert tt.ranks_of(rr)[1:-1] == dense_ranks


def test_truncate_equals_dense_tt_svd_and_error_equality():
    # op = NULL: right-orthonormal remainder => zip-up == TT-SVD of the dense
    # tensor, and ||y - x||^2 = sum delta^2 exactly (SURVEY.md c-A11, A6)
    dims = [2] * 10
    x = rnd(dims, 8, 5)
    xv = tt.to_dense_vector(x)
    for mr, eps in ((4, 0.0), (0, 0.05), (3, 1e-3)):
        r = zipup("truncate", None, x, eps, mr)
        ref, d2 = tt.tt_svd(xv, dims, eps, mr)
        assert r["ranks"] == tt.ranks_of(ref)
        y = tt.to_dense_vector(r["cores"])
        assert np.linalg.norm(y - tt.to_dense_vector(ref)) <= 1e-11 * np.linalg.norm(xv)
        np.testing.assert_allclose(r["delta2"], d2, rtol=1e-9, atol=1e-24)
        err2 = np.sum((y - xv) ** 2)
        assert abs(err2 - sum(r["delta2"])) <= 1e-9 * max(err2, 1e-30) + 1e-24


def _orthogonal(d, rng):
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    return Q


def test_matvec_kron_orthogonal_equals_tt_svd():
    # operator = (x)_q c_q M_q with orthogonal M_q: the exact remainder is an isometry up to
    # scale, so zip-up == TT-SVD of the dense product (catches transposed / mis-indexed W)
    rng = np.random.default_rng(6)
    dims = [2, 3, 2, 2, 3, 2, 2]
    Ms = [1.7 * _orthogonal(d, rng) for d in dims]
    W = [M.reshape(1, d, d, 1) for M, d in zip(Ms, dims)]
    x = rnd(dims, 6, 7)
    Md = Ms[0]
    for M in Ms[1:]:
        Md = np.kron(Md, M)
    yv = Md @ tt.to_dense_vector(x)
    for mr, eps in ((3, 0.0), (0, 0.02)):
        r = zipup("matvec", W, x, eps, mr)
        ref, d2 = tt.tt_svd(yv, dims, eps, mr)
        assert r["ranks"] == tt.ranks_of(ref)
        assert np.linalg.norm(tt.to_dense_vector(r["cores"]) - tt.to_dense_vector(ref)) <= 1e-11 * np.linalg.norm(yv)
    # a transposed operator must give a different result
    Wt = [M.T.reshape(1, d, d, 1) for M, d in zip(Ms, dims)]
    r = zipup("matvec", Wt, x, 0.0, 3)
    assert np.linalg.norm(tt.to_dense_vector(r["cores"]) - tt.to_dense_vector(ref)) > 1e-3


def test_hadamard_sign_train_equals_tt_svd():
    # a rank-1 train with entries +-1: the Hadamard remainder is an isometry, so the
    # zip-up equals the TT-SVD of a*x (catches i/j or operand mix-ups in 'i,i->i')
    rng = np.random.default_rng(8)
    dims = [2] * 9
    a = [rng.choice([-1.0, 1.0], size=(1, 2, 1)) for _ in dims]
    x = rnd(dims, 6, 9)
    yv = tt.to_dense_vector(a) * tt.to_dense_vector(x)
    r = zipup("hadamard", a, x, 0.0, 3)
    ref, d2 = tt.tt_svd(yv, dims, 0.0, 3)
    assert r["ranks"] == tt.ranks_of(ref)
    assert np.linalg.norm(tt.to_dense_vector(r["cores"]) - tt.to_dense_vector(ref)) <= 1e-11 * np.linalg.norm(yv)


def test_identity_operator_equals_truncate():
    dims = [2] * 8
    x = rnd(dims, 8, 10)
    I = gen.identity_mpo(dims).cores
    a = zipup("matvec", I, x, 1e-3, 5)
    b = zipup("truncate", None, x, 1e-3, 5)
    assert a["ranks"] == b["ranks"]
    np.testing.assert_allclose(tt.to_dense_vector(a["cores"]), tt.to_dense_vector(b["cores"]), atol=1e-12)


def test_hadamard_error_bound():
    # ||e||^2 <= sum delta^2 for right-orthonormal states (proof in SURVEY.md §8(c) Pins)
    rng = np.random.default_rng(11)
    for t in range(12):
        a, b = rnd([2] * 10, int(rng.integers(2, 9)), 100 + t), rnd([2] * 10, int(rng.integers(2, 9)), 200 + t)
        mr = int(rng.integers(2, 12))
        r = zipup("hadamard", a, b, 0.0, mr)
        ex = tt.to_dense_vector(a) * tt.to_dense_vector(b)
        e2 = np.sum((tt.to_dense_vector(r["cores"]) - ex) ** 2)
        assert e2 <= sum(r["delta2"]) * (1 + 1e-9) + 1e-24 * np.sum(ex ** 2)


def test_mpo_error_bound_orthonormalized_operator():
    # with every operand right-orthonormalised the plain bound held 700/700;
    # roundoff floor 1e3*eps*||W||_2*||x|| (c-A11)
    rng = np.random.default_rng(12)
    for t in range(10):
        L = int(rng.integers(6, 10))
        dims = [2] * L
        x = rnd(dims, int(rng.integers(2, 9)), 300 + t)
        W = gen.random_mpo(dims, int(rng.integers(2, 5)), np.random.default_rng(400 + t))
        mr = int(rng.integers(1, 10))
        r = zipup("matvec", W.cores, x, 0.0, mr)
        M = dense_op(W)
        xv = tt.to_dense_vector(x)
        e = np.linalg.norm(tt.to_dense_vector(r["cores"]) - M @ xv)
        floor = 1e3 * 2.2e-16 * np.linalg.norm(M, 2) * np.linalg.norm(xv)
        assert e <= math.sqrt(sum(r["delta2"])) * (1 + 1e-9) + floor


def test_prepass_gauge_invariance():
    # pre-pass by QR vs by SVD + random orthogonal gauge -> same result
    dims = [2] * 12
    rng = np.random.default_rng(13)
    B = rnd(dims, 8, 14)
    x = tt.add(B, tt.scale(B, 0.5))                 # redundant rank 16, true rank 8
    W = gen.random_mpo(dims, 3, np.random.default_rng(15)).cores
    r1 = zipup("matvec", W, x, 1e-10, 6)
    # apply random invertible (orthogonal) gauges on every bond of x and W
    def gauge(cores):
        cs = [c.copy() for c in cores]
        for q in range(len(cs) - 1):
            k = cs[q].shape[-1]
            G = _orthogonal(k, rng)
            cs[q] = (cs[q].reshape(-1, k) @ G).reshape(cs[q].shape)
            cs[q + 1] = (G.T @ cs[q + 1].reshape(k, -1)).reshape(cs[q + 1].shape)
        return cs
    r2 = zipup("matvec", gauge(W), gauge(x), 1e-10, 6)
    assert r1["ranks"] == r2["ranks"]
    y1, y2 = tt.to_dense_vector(r1["cores"]), tt.to_dense_vector(r2["cores"])
    assert np.linalg.norm(y1 - y2) <= 1e-12 * np.linalg.norm(y1)


def test_zero_input():
    # SURVEY.md c-A10: all-zero site matrices -> k = 1, zero carry, delta2 = 0
    x = [np.zeros((1, 2, 2)), np.zeros((2, 2, 2)), np.zeros((2, 2, 1))]
    r = zipup("truncate", None, x, 1e-8, 4)
    assert r["ranks"] == [1, 1, 1, 1]
    assert r["delta2"] == [0.0, 0.0]
    assert r["norm"] == 0.0


def test_diff_norm_of_zipup_vs_dense():
    # comparison machinery (c-A29): QR-sweep distance of two trains agrees with dense
    dims = [2] * 12
    x = rnd(dims, 8, 16)
    W = gen.random_mpo(dims, 3, np.random.default_rng(17)).cores
    a = zipup("matvec", W, x, 1e-6, 12)["cores"]
    b = zipup("matvec", W, x, 1e-6, 10)["cores"]
    d = np.linalg.norm(tt.to_dense_vector(a) - tt.to_dense_vector(b))
    assert abs(tt.diff_norm(a, b) - d) <= 1e-10 * np.linalg.norm(tt.to_dense_vector(a))
