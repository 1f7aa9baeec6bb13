"""Tensorized discrete Fourier transform by a chain of Hadamard zip-ups, §4
"Fourier transformation" (lines 533-566) -- SURVEY.md §8(f) row f2.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  M(i, j) = v^(i j), v = exp(-2 pi i / N)
  M = prod_q T(i_q, j) element-wise, each T(i_q, .) a rank-b_q train
  "This multiplication can be done with a zip-up algorithm"

The factors come from ``paper_2602_20226_b200.gen.qft_trains`` (inputs, no zip-up
arithmetic).  Reading (DESIGN.md c-A34): the chain is Y_1 = T_1, Y_q = zip-up(T_q o Y_{q-1})
for q = 2..n with the given max rank and eps = 0 (the paper quotes maximum ranks only); the
distance of PAPER.md:566 is the Frobenius norm ||M - Y_n||_F.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

from .tt import full_legs
from .zipup import zipup


def dft_matrix(N: int) -> np.ndarray:
    """M(i, j) = exp(-2 pi i (i j mod N) / N), the exponent reduced in integers."""
    i = np.arange(N, dtype=np.int64)
    e = np.outer(i, i) % N
    return np.exp(-2j * np.pi * e / N)


def chain(trains: Sequence[Sequence[np.ndarray]], max_rank: int, eps: float = 0.0) -> List[np.ndarray]:
    y = [np.asarray(c) for c in trains[0]]
    for t in trains[1:]:
        y = zipup("hadamard", t, y, eps, max_rank)["cores"]
    return y


def to_matrix(cores, bases_i: Sequence[int]) -> np.ndarray:
    """Dense N x N matrix of a train in the QFT digit layout (rows i, columns j)."""
    from paper_2602_20226_b200.gen import qft_dense_order
    shape, perm = qft_dense_order(bases_i)
    N = int(np.prod(bases_i))
    return full_legs(cores).reshape(shape).transpose(perm).reshape(N, N)


def distance(cores, bases_i: Sequence[int]) -> float:
    """||M - Y||_F against the exact DFT matrix."""
    N = int(np.prod(bases_i))
    return float(np.linalg.norm(to_matrix(cores, bases_i) - dft_matrix(N)))
