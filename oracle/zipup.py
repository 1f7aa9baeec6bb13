"""Zip-up (decomposition) algorithm, §3.2 (lines 253-275), window N = 1.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Follows the paper's order:

  1. "the tensor trains that are part of the operation shift their normalization
     center to the left end"  -> right_orthonormalize every operand,
     the MPO included as a TT over (d_out*d_in) (SURVEY.md c-A2).
  2. "the first N-cores ... are contracted exactly according to some calculation rule"
     (Eq. einsum) -> site matrix T_q with rows (chi, i)
     and columns (w', r') (xi = mu nu).
  3. "splitting C(i_1..i_N) into C(i_1) C(i_2..i_N) with some kind of approximate matrix
     decomposition" -- the SVD of Fig. decomposition_algorithm
      -- here LAPACK gesdd applied directly to T_q, truncated by the rule
     of SPEC.md:299 (oracle.tt.truncation_rank).
  4. the left factor U_k is the output core (left-orthonormal, so no normalisation
     restore is needed, SURVEY.md c-A6); the remainder diag(s_k) Vh_k is carried and
     "extended ... using A(i_{N+1}) and B(i_{N+1})".
  5. "repeated until no more cores can be added, after which the super-core is fully
     decomposed": the last T is the last core (SURVEY.md c-A7).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from .tt import right_orthonormalize, tail_sum, truncation_rank


def _svd(M: np.ndarray):
    try:
        return np.linalg.svd(M, full_matrices=False)
    except np.linalg.LinAlgError:  # gesdd did not converge: fall back to gesvd
        import scipy.linalg
        return scipy.linalg.svd(M, full_matrices=False, lapack_driver="gesvd")


def site_matrix(kind: str, G: np.ndarray, Xq: np.ndarray, Oq: Optional[np.ndarray]) -> np.ndarray:
    """Exact local contraction of the carry G (chi, w, r) with the operand cores
    (Eq. einsum).  Returns T (chi, i, w', r')."""
    # optimize=True: numpy evaluates the same sum pairwise (G with the state core first) instead
    # of one nested loop over all six indices -- the definition is unchanged, only the order of
    # the floating-point additions; without it a cfg3 site (256^5 x 2 terms) takes tens of minutes
    if kind == "matvec":     # 'ij,j->i': sum over r and j, w
        return np.einsum("cwr,rjs,wijv->civs", G, Xq, Oq, optimize=True)
    if kind == "hadamard":   # 'i,i->i': i shared, not summed
        return np.einsum("cab,bis,aiv->civs", G, Xq, Oq, optimize=True)
    if kind == "truncate":   # identity operation (PAPER.md:710 truncate)
        return np.einsum("cr,ris->cis", G[:, 0, :], Xq)[:, :, None, :]
    raise ValueError(kind)


def zipup(kind: str, op: Optional[Sequence[np.ndarray]], x: Sequence[np.ndarray], eps: float,
          max_rank: int, orth_operator: bool = True, force_ranks: Optional[Sequence[int]] = None,
          on_site=None):
    """on_site(q): optional progress hook called after site q is finished (instrumentation
    only -- bench.py's bounded CPU baseline stops a long run by raising from it).
    Returns a dict with
      cores   : output cores C_q (chi_q, d_q, chi_{q+1})
      ranks   : [1, chi_1, ..., chi_{L-1}, 1]
      delta2  : discarded sum of squares per split (L-1 values)
      sigmas  : singular values of every T_q (q < L-1), descending
      norm    : ||y||_F = ||C_{L-1}||_F (left-canonical output)
    """
    # float64, or complex128 when an operand is complex (the Fourier chain);
    # every step below is written for both (M^T = QR gives right-orthonormal rows in the
    # complex sense too: Q^T conj(Q) = conj(Q^H Q) = I; the SVD carry is diag(s) V^H)
    cplx = any(np.iscomplexobj(c) for c in x) or (op is not None and any(np.iscomplexobj(c) for c in op))
    dt = np.complex128 if cplx else np.float64
    X = right_orthonormalize([np.asarray(c, dtype=dt) for c in x])                # step 1
    if kind == "truncate":
        O = None
    else:
        O = [np.asarray(c, dtype=dt) for c in op]
        if orth_operator:
            O = right_orthonormalize(O)
    L = len(X)
    G = np.ones((1, 1, 1), dtype=dt)          # carry (chi, w, r)
    cores: List[np.ndarray] = []
    delta2: List[float] = []
    sigmas: List[np.ndarray] = []
    ranks = [1]
    for q in range(L):
        T = site_matrix(kind, G, X[q], None if O is None else O[q])              # step 2
        chi, d, v, s = T.shape
        M = T.reshape(chi * d, v * s)
        if q == L - 1:                                                            # step 5
            cores.append(T.reshape(chi, d, 1))
            ranks.append(1)
            break
        U, sig, Vh = _svd(M)                                                      # step 3
        if float(np.sum(sig * sig)) == 0.0:
            # all-zero site matrix (SPEC.md:324 / SURVEY.md c-A10): k = 1, U e_0, zero carry
            k = 1
            U = np.zeros((M.shape[0], 1)); U[0, 0] = 1.0
            sig = np.zeros(1); Vh = np.zeros((1, M.shape[1]))
        else:
            k = truncation_rank(sig, eps, max_rank)
        if force_ranks is not None:
            k = int(force_ranks[q + 1])
        delta2.append(tail_sum(sig, k))
        sigmas.append(sig.copy())
        cores.append(U[:, :k].reshape(chi, d, k))                                 # step 4
        G = (sig[:k, None] * Vh[:k]).reshape(k, v, s)
        ranks.append(k)
        if on_site is not None:
            on_site(q)
    norm = float(np.linalg.norm(cores[-1]))
    return {"cores": cores, "ranks": ranks, "delta2": delta2, "sigmas": sigmas, "norm": norm}


def _absorb(kind: str, C: np.ndarray, Xq: np.ndarray, Oq: Optional[np.ndarray]) -> np.ndarray:
    """Extend the super-core C (chi, P, w, r) -- P the flattened physical indices of the
    pending sites -- by one site, exactly (Eq. einsum): returns
    (chi, P, i, w', r')."""
    if kind == "matvec":
        return np.einsum("cpwr,rjs,wijv->cpivs", C, Xq, Oq, optimize=True)
    if kind == "hadamard":
        return np.einsum("cpab,bis,aiv->cpivs", C, Xq, Oq, optimize=True)
    if kind == "truncate":
        return np.einsum("cpr,ris->cpis", C[:, :, 0, :], Xq)[:, :, :, None, :]
    raise ValueError(kind)


def zipup_window(kind: str, op: Optional[Sequence[np.ndarray]], x: Sequence[np.ndarray], eps: float,
                 max_rank: int, window: int, orth_operator: bool = True,
                 force_ranks: Optional[Sequence[int]] = None):
    """Zip-up with a super-core of N = `window` sites ("the first N-cores
    (1 <= N <= n) are contracted exactly").  Same return dict as zipup().

      1. right-orthonormalise the operands
      2. contract the first N sites exactly into the super-core S (chi=1, i_0..i_{N-1}, w, r)
      3. split S (rows (chi, i_first), columns the rest) by SVD, truncated by the rule of
         SPEC.md:299 and (reading c-A35) by k <= w_{q+1} r_{q+1}, the exact rank of the product
         at that bond; emit U_k; the carry diag(s_k) V_k^H keeps the pending physical indices
         
      4. extend the carry by the next site and repeat
      5. when no site is left, the super-core is "fully decomposed": the same
         split repeated until one physical index remains, which is the last core.
    window = 1 reproduces zipup(); window = L is the exact product followed by TT-SVD
    (SPEC.md:394-396).
    """
    N = int(window)
    cplx = any(np.iscomplexobj(c) for c in x) or (op is not None and any(np.iscomplexobj(c) for c in op))
    dt = np.complex128 if cplx else np.float64
    X = right_orthonormalize([np.asarray(c, dtype=dt) for c in x])                # step 1
    O = None
    if kind != "truncate":
        O = [np.asarray(c, dtype=dt) for c in op]
        if orth_operator:
            O = right_orthonormalize(O)
    L = len(X)
    N = max(1, min(N, L))
    bond = []                                  # w_q * r_q of the exact product at bond q
    for q in range(L + 1):
        rx = X[q].shape[0] if q < L else 1
        ro = (O[q].shape[0] if q < L else 1) if O is not None else 1
        bond.append(rx * ro)
    S = np.ones((1, 1, 1, 1), dtype=dt)        # (chi, P, w, r) with P = 1 (no pending site)
    dims: List[int] = []                       # digit sizes of the pending sites
    nxt = 0
    while nxt < N:                                                                 # step 2
        S = _absorb(kind, S, X[nxt], None if O is None else O[nxt])
        dims.append(X[nxt].shape[1] if kind != "matvec" else O[nxt].shape[1])
        S = S.reshape(S.shape[0], -1, S.shape[-2], S.shape[-1])
        nxt += 1
    cores: List[np.ndarray] = []
    delta2: List[float] = []
    sigmas: List[np.ndarray] = []
    ranks = [1]
    q = 0
    while True:
        chi = S.shape[0]
        if q == L - 1:                          # one physical index left: the last core
            cores.append(S.reshape(chi, dims[0], 1))
            ranks.append(1)
            break
        d0 = dims[0]
        M = S.reshape(chi * d0, -1)                                                # step 3
        U, sig, Vh = _svd(M)
        if float(np.sum(np.abs(sig) ** 2)) == 0.0:
            k = 1
            U = np.zeros((M.shape[0], 1), dtype=dt); U[0, 0] = 1.0
            sig = np.zeros(1); Vh = np.zeros((1, M.shape[1]), dtype=dt)
        else:
            k = truncation_rank(sig, eps, max_rank)
            k = min(k, bond[q + 1])              # c-A35
        if force_ranks is not None:
            k = int(force_ranks[q + 1])
        delta2.append(tail_sum(sig, k))
        sigmas.append(sig.copy())
        cores.append(U[:, :k].reshape(chi, d0, k))
        rest = S.shape[2:]                      # (w, r)
        dims = dims[1:]
        S = (sig[:k, None] * Vh[:k]).reshape((k, int(np.prod(dims)) if dims else 1) + rest)
        ranks.append(k)
        q += 1
        if nxt < L:                                                                # step 4
            S = _absorb(kind, S, X[nxt], None if O is None else O[nxt])
            dims.append(X[nxt].shape[1] if kind != "matvec" else O[nxt].shape[1])
            S = S.reshape(S.shape[0], -1, S.shape[-2], S.shape[-1])
            nxt += 1
    norm = float(np.linalg.norm(cores[-1]))
    return {"cores": cores, "ranks": ranks, "delta2": delta2, "sigmas": sigmas, "norm": norm}
