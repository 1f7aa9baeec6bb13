"""Variational refinement seeded by the zip-up, §3.3 "Variational algorithms"
(lines 277-301) -- SURVEY.md §8(f) row f3.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  |C - O(A, B)| -> min; with C(i_q) the normalisation centre
  C(i_q) = d<C|O(A, B)> / dC*(i_q)                           (Eq. variational)
  "the start is to the left and the cores are optimized sequentially by going to the right
   and back again.  A good starting guess for C is the result of the decomposition approach"
                                                             

Single-site version (reading c-A36): C is right-orthonormalised (centre at site 0); a sweep
updates sites 0..L-1 (after each update a QR moves the centre right) and then L-1..0 (an LQ
moves it left); bond ranks stay those of the seed.  With the centre at q, <C|C> = |C_q|^2
and the update maximises it, so |O - C|^2 = |O|^2 - |C_q|^2 never increases.  Real trains.

Two-site version, ncores = 2 ("By fusing multiple adjacent C(i_q) into a
super-core C(i_q,...,i_{q+N}) and solving (Eq. variational) with it, it is possible to realize
multi-core strategies, which normally leads to better convergence and an efficient way of
controlling the ranks of the cores.  After the optimization C(i_q,...,i_{q+N}) can be again
fully decomposed"; the paper's own call is variational(max_rank=8, cutoff=0.0, ncores=2,
nsweeps=2); reading c-A37): the super-core of sites (q, q+1) is
S = d<C|O>/dS* = Le[q] W_q x_q W_{q+1} x_{q+1} Re[q+2]; it is decomposed by an SVD of its
(c d_q) x (d_{q+1} a) matricisation truncated by the zip-up's rule (SPEC.md:299 with
eps = cutoff, k <= max_rank).  Sweeping right (q = 0..L-2) C_q = U_k and the centre
diag(s_k) V_k^T moves to q+1; sweeping back (q = L-2..0) C_{q+1} = V_k^T and C_q = U_k diag(s_k).
The recorded quantity is |S_k|^2 = sum_{j<=k} s_j^2 (the centre's norm after the split);
ranks adapt between sweeps.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from .tt import right_orthonormalize, truncation_rank


def _opcore(kind: str, Oq: Optional[np.ndarray], d: int) -> np.ndarray:
    """The operator core as W[w, i, j, w'] (Hadamard: A[w, i, w'] on the diagonal i == j;
    truncate: the identity with w = w' = 1)."""
    if kind == "matvec":
        return Oq
    if kind == "hadamard":
        w, dd, w2 = Oq.shape
        W = np.zeros((w, dd, dd, w2))
        for i in range(dd):
            W[:, i, i, :] = Oq[:, i, :]
        return W
    return np.eye(d).reshape(1, d, d, 1)


def variational(kind: str, op: Optional[Sequence[np.ndarray]], x: Sequence[np.ndarray],
                seed: Sequence[np.ndarray], sweeps: int, ncores: int = 1, eps: float = 0.0,
                max_rank: int = 0):
    """Returns {"cores": C (centre at site 0), "center_norm2": [|C_q|^2 (ncores = 1) or the
    truncated super-core's |S_k|^2 (ncores = 2) after every update], "ranks"}.
    eps / max_rank: the split's truncation (ncores = 2 only)."""
    if ncores == 2:
        return _variational2(kind, op, x, seed, sweeps, eps, max_rank)
    if ncores != 1:
        raise ValueError("ncores must be 1 or 2")
    X = [np.asarray(c, dtype=np.float64) for c in x]
    L = len(X)
    W = [_opcore(kind, None if op is None else np.asarray(op[q], dtype=np.float64), X[q].shape[1])
         for q in range(L)]
    C = right_orthonormalize([np.asarray(c, dtype=np.float64) for c in seed])
    # environments: Le[q] = (c, w, r) from the left of site q, Re[q] from the right of site q-1
    Le: List[Optional[np.ndarray]] = [None] * (L + 1)
    Re: List[Optional[np.ndarray]] = [None] * (L + 1)
    Le[0] = np.ones((1, 1, 1))
    Re[L] = np.ones((1, 1, 1))
    for q in range(L - 1, 0, -1):
        Re[q] = np.einsum("cia,wijv,rjs,avs->cwr", C[q], W[q], X[q], Re[q + 1], optimize=True)
    norms = []

    def update(q):
        C[q] = np.einsum("cwr,wijv,rjs,avs->cia", Le[q], W[q], X[q], Re[q + 1], optimize=True)  # Eq. variational
        norms.append(float(np.sum(C[q] * C[q])))

    for _ in range(sweeps):
        for q in range(L):                                   # to the right
            update(q)
            if q < L - 1:
                c, d, a = C[q].shape
                Q, R = np.linalg.qr(C[q].reshape(c * d, a))
                C[q] = Q.reshape(c, d, Q.shape[1])
                C[q + 1] = np.einsum("ab,bis->ais", R, C[q + 1], optimize=True)
                Le[q + 1] = np.einsum("cia,cwr,wijv,rjs->avs", C[q], Le[q], W[q], X[q], optimize=True)
        for q in range(L - 1, -1, -1):                       # and back
            update(q)
            if q > 0:
                c, d, a = C[q].shape
                Q, R = np.linalg.qr(C[q].reshape(c, d * a).T)   # C_q = R^T Q^T
                C[q] = Q.T.reshape(Q.shape[1], d, a)
                C[q - 1] = np.einsum("cia,ab->cib", C[q - 1], R.T, optimize=True)
                Re[q] = np.einsum("cia,wijv,rjs,avs->cwr", C[q], W[q], X[q], Re[q + 1], optimize=True)
    return {"cores": C, "center_norm2": norms, "ranks": [int(C[0].shape[0])] + [int(c.shape[-1]) for c in C]}


def _variational2(kind, op, x, seed, sweeps, eps, max_rank):
    """Two-site sweeps (see the module docstring; reading c-A37)."""
    X = [np.asarray(c, dtype=np.float64) for c in x]
    L = len(X)
    if L < 2:
        raise ValueError("ncores = 2 needs at least two sites")
    W = [_opcore(kind, None if op is None else np.asarray(op[q], dtype=np.float64), X[q].shape[1])
         for q in range(L)]
    C = right_orthonormalize([np.asarray(c, dtype=np.float64) for c in seed])
    Le: List[Optional[np.ndarray]] = [None] * (L + 1)
    Re: List[Optional[np.ndarray]] = [None] * (L + 1)
    Le[0] = np.ones((1, 1, 1))
    Re[L] = np.ones((1, 1, 1))

    def right_env(q):
        Re[q] = np.einsum("cia,wijv,rjs,avs->cwr", C[q], W[q], X[q], Re[q + 1], optimize=True)

    def left_env(q):                             # Le[q+1] from the left-orthonormal C_q
        Le[q + 1] = np.einsum("cia,cwr,wijv,rjs->avs", C[q], Le[q], W[q], X[q], optimize=True)

    for q in range(L - 1, 1, -1):
        right_env(q)
    norms = []

    def split(q):
        # S[c, i, k, a] = Le[q] W_q x_q W_{q+1} x_{q+1} Re[q+2]        (Eq. variational, N = 2)
        S = np.einsum("cwr,wijv,rjs,vklu,slt,aut->cika", Le[q], W[q], X[q], W[q + 1], X[q + 1], Re[q + 2],
                      optimize=True)
        c, d1, d2, a = S.shape
        U, sig, Vh = np.linalg.svd(S.reshape(c * d1, d2 * a), full_matrices=False)
        k = truncation_rank(sig, eps, max_rank)
        norms.append(float(np.sum(sig[:k] ** 2)))
        return U[:, :k].reshape(c, d1, k), sig[:k], Vh[:k].reshape(k, d2, a)

    for _ in range(sweeps):
        for q in range(L - 1):                   # to the right: centre moves to q+1
            U, sg, V = split(q)
            C[q] = U
            C[q + 1] = sg[:, None, None] * V
            left_env(q)
        for q in range(L - 2, -1, -1):           # and back: centre moves to q
            U, sg, V = split(q)
            C[q + 1] = V
            C[q] = U * sg[None, None, :]
            right_env(q + 1)
    return {"cores": C, "center_norm2": norms, "ranks": [1] + [int(c.shape[-1]) for c in C]}
