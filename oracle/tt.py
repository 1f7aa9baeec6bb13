"""Exact tensor-train algebra in float64 (oracle; test infrastructure only).

Each function cites the passage it follows.  Cores are numpy arrays:
MPS (r, d, r'), MPO (w, d_out, d_in, w').  Digits big-endian.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence

import numpy as np


# ------------------------------------------------------------------------------ dense

def _legs(core):
    return core.shape[1:-1]


def full_legs(cores: Sequence[np.ndarray]) -> np.ndarray:
    """Contract all cores (Eq. vector_dec / tensor_dec) into one array
    with axes (legs of site 0, legs of site 1, ...), bonds summed."""
    acc = np.ones((1, 1))  # (flattened legs so far, bond)
    leg_shape: List[int] = []
    for c in cores:
        r = c.shape[0]
        legs = _legs(c)
        acc = acc @ c.reshape(r, -1)  # (legs_so_far, legs*r')
        acc = acc.reshape(-1, c.shape[-1])
        leg_shape.extend(legs)
    assert acc.shape[1] == 1, "last bond must be 1"
    return acc.reshape(leg_shape)


def _dim_order(leg_dim: Optional[Sequence[int]], L: int) -> List[int]:
    if leg_dim is None:
        return list(range(L))
    order = []
    for dim in sorted(set(leg_dim)):
        order.extend([q for q in range(L) if leg_dim[q] == dim])
    return order


def to_dense_vector(cores, leg_dim=None) -> np.ndarray:
    """Dense vector over the original dimensions, row-major (dimension 0 slowest),
    digits of each dimension most significant first."""
    T = full_legs(cores)
    order = _dim_order(leg_dim, len(cores))
    return np.ascontiguousarray(T.transpose(order)).reshape(-1)


def to_dense_matrix(cores, leg_dim=None) -> np.ndarray:
    """Dense operator M[out, in] for an MPO (legs (d_out, d_in) per site)."""
    L = len(cores)
    T = full_legs(cores)  # axes: o0, i0, o1, i1, ...
    order = _dim_order(leg_dim, L)
    perm = [2 * q for q in order] + [2 * q + 1 for q in order]
    n_out = math.prod(c.shape[1] for c in cores)
    n_in = math.prod(c.shape[2] for c in cores)
    return np.ascontiguousarray(T.transpose(perm)).reshape(n_out, n_in)


def evaluate(cores, digits: np.ndarray) -> np.ndarray:
    """Entries at multi-indices digits[n, L] (one digit per site): product of the selected
    core slices.  MPS only."""
    digits = np.asarray(digits)
    n = digits.shape[0]
    v = np.ones((n, 1))
    for q, c in enumerate(cores):
        sl = c[:, digits[:, q], :]           # (r, n, r')
        v = np.einsum("na,anb->nb", v, sl)
    return v[:, 0]


# ------------------------------------------------------------------------ exact ops

def inner(a, b):
    """<a, b> = sum_i conj(a_i) b_i by a left-to-right environment sweep,
    conjugate-linear in the first argument.  Returns a float for real trains
    and a complex for complex ones."""
    E = np.ones((1, 1))
    for x, y in zip(a, b):
        rx, ry = x.shape[0], y.shape[0]
        X = np.conj(x.reshape(rx, -1, x.shape[-1]))
        Y = y.reshape(ry, -1, y.shape[-1])
        E = np.einsum("ab,aic,bid->cd", E, X, Y)
    v = E[0, 0]
    return complex(v) if np.iscomplexobj(E) else float(v)


def add(a, b) -> List[np.ndarray]:
    """Exact addition by block cores: first core [A B], middle cores
    diag(A, B), last core [A; B].  Ranks add."""
    L = len(a)
    if L == 1:
        return [a[0] + b[0]]
    out = []
    for q in range(L):
        A, B = a[q], b[q]
        if q == 0:
            out.append(np.concatenate([A, B], axis=-1))
        elif q == L - 1:
            out.append(np.concatenate([A, B], axis=0))
        else:
            C = np.zeros((A.shape[0] + B.shape[0],) + _legs(A) + (A.shape[-1] + B.shape[-1],),
                         dtype=np.result_type(A, B))
            C[: A.shape[0], ..., : A.shape[-1]] = A
            C[A.shape[0]:, ..., A.shape[-1]:] = B
            out.append(C)
    return out


def scale(a, s) -> List[np.ndarray]:
    out = [c.copy() for c in a]
    out[0] = out[0] * s
    return out


def exact_matvec(W, x) -> List[np.ndarray]:
    """Exact 'ij,j->i' by the local summation of Eq. einsum:
    C_q[(w,r), i, (w',r')] = sum_j W_q[w,i,j,w'] x_q[r,j,r'] (bond flatten xi = mu nu)."""
    out = []
    for Wq, xq in zip(W, x):
        w, di, dj, w2 = Wq.shape
        r, dj2, r2 = xq.shape
        assert dj == dj2
        C = np.einsum("aijb,cjd->acibd", Wq, xq).reshape(w * r, di, w2 * r2)
        out.append(C)
    return out


def exact_hadamard(a, b) -> List[np.ndarray]:
    """Exact 'i,i->i' (element-wise product) by Eq. einsum with the digit shared, not
    summed: C_q[(a,b), i, (a',b')] = a_q[a,i,a'] b_q[b,i,b'] (ranks multiply)."""
    out = []
    for A, B in zip(a, b):
        ra, d, ra2 = A.shape
        rb, d2, rb2 = B.shape
        assert d == d2
        out.append(np.einsum("aic,bid->abicd", A, B).reshape(ra * rb, d, ra2 * rb2))
    return out


def exact_matmat(A, B) -> List[np.ndarray]:
    """Exact 'ij,jk->ik' of two MPOs by Eq. einsum."""
    out = []
    for Aq, Bq in zip(A, B):
        a, di, dj, a2 = Aq.shape
        b, dj2, dk, b2 = Bq.shape
        out.append(np.einsum("aijc,bjkd->abikcd", Aq, Bq).reshape(a * b, di, dk, a2 * b2))
    return out


# --------------------------------------------------------------- normalisation (QR)

def _unfold_left(c):
    return c.reshape(c.shape[0], -1)


def right_orthonormalize(cores) -> List[np.ndarray]:
    """Shift the normalisation centre to the left end by thin QR
    ("for example using a QR decomposition"):
    for q = L-1..1: core_q^T = Q R, core_q <- Q^T, core_{q-1} <- core_{q-1} x_last R^T.
    Legs of an MPO core are treated as one (d_out*d_in) leg (SURVEY.md c-A2)."""
    cs = [c.copy() for c in cores]
    for q in range(len(cs) - 1, 0, -1):
        c = cs[q]
        legs = _legs(c)
        M = _unfold_left(c)                   # (r_q, legs*r')
        Q, R = np.linalg.qr(M.T)              # M^T = Q R, Q: (legs*r', k)
        k = Q.shape[1]
        cs[q] = Q.T.reshape((k,) + legs + (c.shape[-1],))
        p = cs[q - 1]
        cs[q - 1] = (p.reshape(-1, p.shape[-1]) @ R.T).reshape(p.shape[:-1] + (k,))
    return cs


def left_orthonormalize(cores) -> List[np.ndarray]:
    """Mirror image: centre at the right end."""
    cs = [c.copy() for c in cores]
    for q in range(len(cs) - 1):
        c = cs[q]
        M = c.reshape(-1, c.shape[-1])
        Q, R = np.linalg.qr(M)
        k = Q.shape[1]
        cs[q] = Q.reshape(c.shape[:-1] + (k,))
        n = cs[q + 1]
        cs[q + 1] = (R @ n.reshape(n.shape[0], -1)).reshape((k,) + n.shape[1:])
    return cs


def qr_norm(cores) -> float:
    """Frobenius norm by a left-to-right QR sweep: after left-orthonormalisation the norm
    lives in the last core.  Resolves tiny differences that the
    Gram identity cannot."""
    cs = left_orthonormalize(cores)
    return float(np.linalg.norm(cs[-1]))


def diff_norm(x, y) -> float:
    """||x - y||_F via the exact block sum x + (-1) y and a QR sweep."""
    return qr_norm(add(x, scale(y, -1.0)))


def is_left_orthonormal(c, tol=1e-12) -> bool:
    M = c.reshape(-1, c.shape[-1])
    return np.allclose(M.T @ M, np.eye(M.shape[1]), atol=tol)


def is_right_orthonormal(c, tol=1e-12) -> bool:
    M = c.reshape(c.shape[0], -1)
    return np.allclose(M @ M.T, np.eye(M.shape[0]), atol=tol)


# ------------------------------------------------------------------- truncation

def truncation_rank(sig: np.ndarray, eps: float, max_rank: int) -> int:
    """SPEC.md:299 (SURVEY.md a5 / c-A4): k = min(max_rank, smallest k>=1 with
    sqrt(sum_{j>k} s_j^2) <= eps * sqrt(sum_j s_j^2)); tails summed smallest first;
    k = 1 for an all-zero spectrum; max_rank <= 0 means unbounded."""
    sig = np.asarray(sig, dtype=np.float64)
    p = sig.size
    s2 = sig * sig
    tot = float(s2.sum())
    if tot == 0.0:
        return 1
    tail = np.zeros(p + 1)
    acc = 0.0
    for j in range(p - 1, -1, -1):   # tail[j] = sum_{i>=j} s_i^2, smallest first
        acc += s2[j]
        tail[j] = acc
    tau = (eps * eps) * tot
    k = p
    for kk in range(1, p + 1):
        if tail[kk] <= tau:
            k = kk
            break
    if max_rank > 0:
        k = min(k, max_rank)
    return max(1, k)


def tail_sum(sig: np.ndarray, k: int) -> float:
    s2 = np.asarray(sig, dtype=np.float64) ** 2
    acc = 0.0
    for j in range(s2.size - 1, k - 1, -1):
        acc += s2[j]
    return acc


# ------------------------------------------------------------------- TT-SVD / round

def tt_svd(dense: np.ndarray, dims: Sequence[int], eps: float, max_rank: int):
    """Left-to-right sequential truncated SVD of a dense vector (Oseledets TT-SVD) with
    the per-split rule of SPEC.md:299.  Returns (cores, delta2 per split)."""
    L = len(dims)
    M = np.asarray(dense, dtype=np.float64).reshape(1, -1)
    cores, d2 = [], []
    r = 1
    for q in range(L - 1):
        M = M.reshape(r * dims[q], -1)
        U, s, Vh = np.linalg.svd(M, full_matrices=False)
        k = truncation_rank(s, eps, max_rank)
        d2.append(tail_sum(s, k))
        cores.append(U[:, :k].reshape(r, dims[q], k))
        M = s[:k, None] * Vh[:k]
        r = k
    cores.append(M.reshape(r, dims[L - 1], 1))
    return cores, d2


def round_train(cores, eps: float, max_rank: int):
    """Rounding (PAPER.md:710 ``truncate``): left-orthonormalise by QR, then
    a right-to-left truncated-SVD sweep with the SPEC.md:299 rule."""
    cs = left_orthonormalize(cores)
    for q in range(len(cs) - 1, 0, -1):
        c = cs[q]
        M = c.reshape(c.shape[0], -1)
        U, s, Vh = np.linalg.svd(M, full_matrices=False)
        k = truncation_rank(s, eps, max_rank)
        cs[q] = Vh[:k].reshape((k,) + c.shape[1:])
        p = cs[q - 1]
        cs[q - 1] = (p.reshape(-1, p.shape[-1]) @ (U[:, :k] * s[:k])).reshape(p.shape[:-1] + (k,))
    return cs


def ranks_of(cores) -> List[int]:
    return [int(cores[0].shape[0])] + [int(c.shape[-1]) for c in cores]
