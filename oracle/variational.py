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
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from .tt import right_orthonormalize


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
                seed: Sequence[np.ndarray], sweeps: int):
    """Returns {"cores": C (centre at site 0), "center_norm2": [|C_q|^2 after every update]}."""
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
        Re[q] = np.einsum("cia,wijv,rjs,avs->cwr", C[q], W[q], X[q], Re[q + 1])
    norms = []

    def update(q):
        C[q] = np.einsum("cwr,wijv,rjs,avs->cia", Le[q], W[q], X[q], Re[q + 1])     # Eq. variational
        norms.append(float(np.sum(C[q] * C[q])))

    for _ in range(sweeps):
        for q in range(L):                                   # to the right
            update(q)
            if q < L - 1:
                c, d, a = C[q].shape
                Q, R = np.linalg.qr(C[q].reshape(c * d, a))
                C[q] = Q.reshape(c, d, Q.shape[1])
                C[q + 1] = np.einsum("ab,bis->ais", R, C[q + 1])
                Le[q + 1] = np.einsum("cia,cwr,wijv,rjs->avs", C[q], Le[q], W[q], X[q])
        for q in range(L - 1, -1, -1):                       # and back
            update(q)
            if q > 0:
                c, d, a = C[q].shape
                Q, R = np.linalg.qr(C[q].reshape(c, d * a).T)   # C_q = R^T Q^T
                C[q] = Q.T.reshape(Q.shape[1], d, a)
                C[q - 1] = np.einsum("cia,ab->cib", C[q - 1], R.T)
                Re[q] = np.einsum("cia,wijv,rjs,avs->cwr", C[q], W[q], X[q], Re[q + 1])
    return {"cores": C, "center_norm2": norms}
