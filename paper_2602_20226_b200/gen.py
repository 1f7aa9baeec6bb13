"""Seeded synthetic inputs for the zip-up hot path (BASELINE.json ``configs[0..4]``).

This module is shared by the CPU oracle (``oracle/``), the GPU parity tests and
``bench.py``.  It holds NO zip-up arithmetic: it only draws random cores and
writes out the paper's closed-form structured trains (§4) as arrays.
Every structured train built here is pinned against its dense definition in
``tests/test_gen.py``.

Conventions:
  * MPS core  q: shape (r_q, d_q, r_{q+1})            row-major, leftmost slowest
  * MPO core  q: shape (w_q, d_out_q, d_in_q, w_{q+1})
  * digits are big-endian: core 0 carries the most significant digit,
    c_q = prod_{r>q} b_r (Eq. quantization).
  * seeds: numpy PCG64(SeedSequence([2602, cfg, member, operand])),
    cores drawn in site order, ``standard_normal(shape)`` in C order, then scaled.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

SEED_ROOT = 2602


def rng_for(cfg: int, member: int, operand: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED_ROOT, cfg, member, operand])))


def digit_factors(bases: Sequence[int]) -> List[int]:
    """c_q = prod_{r>q} b_r."""
    c = [1] * len(bases)
    for q in range(len(bases) - 2, -1, -1):
        c[q] = c[q + 1] * bases[q + 1]
    return c


def clipped_ranks(dims: Sequence[int], R: int) -> List[int]:
    """Uniform bond rank R clipped by the unfolding sizes (SURVEY.md c-A13):
    r_q = min(R, prod_{s<q} d_s, prod_{s>=q} d_s), r_0 = r_L = 1."""
    L = len(dims)
    out = []
    for q in range(L + 1):
        left = math.prod(dims[:q])
        right = math.prod(dims[q:])
        out.append(int(min(R, left, right)))
    return out


@dataclass
class Train:
    """A tensor train as a list of numpy cores plus the digit layout.

    ``leg_dim[q]`` names the original dimension that site q's digit belongs to
    (digits of one dimension appear in order, most significant first).
    """
    cores: List[np.ndarray]
    kind: str = "mps"              # "mps" | "mpo"
    leg_dim: Optional[List[int]] = None

    @property
    def L(self) -> int:
        return len(self.cores)

    @property
    def ranks(self) -> List[int]:
        return [int(self.cores[0].shape[0])] + [int(c.shape[-1]) for c in self.cores]

    @property
    def dims(self) -> List[int]:
        return [int(c.shape[1]) for c in self.cores]

    def astype(self, dt) -> "Train":
        return Train([np.ascontiguousarray(c.astype(dt)) for c in self.cores], self.kind,
                     None if self.leg_dim is None else list(self.leg_dim))


# --------------------------------------------------------------------------------------
# random trains
# --------------------------------------------------------------------------------------

def random_mps(dims: Sequence[int], R: int, rng: np.random.Generator, std: float = 1.0,
               ranks: Optional[Sequence[int]] = None) -> Train:
    r = list(ranks) if ranks is not None else clipped_ranks(dims, R)
    cores = []
    for q, d in enumerate(dims):
        cores.append(rng.standard_normal((r[q], d, r[q + 1])) * std)
    return Train(cores, "mps")


def random_mpo(dims: Sequence[int], R: int, rng: np.random.Generator, std: float = 1.0) -> Train:
    """Random MPO with bonds min(R, prod_{s<q} d_s^2, prod_{s>=q} d_s^2)."""
    sq = [d * d for d in dims]
    w = clipped_ranks(sq, R)
    cores = []
    for q, d in enumerate(dims):
        cores.append(rng.standard_normal((w[q], d, d, w[q + 1])) * std)
    return Train(cores, "mpo")


def env_norm(t: Train) -> float:
    """Frobenius norm of an MPS by a left environment sweep (input preparation only)."""
    E = np.ones((1, 1))
    for c in t.cores:
        E = np.einsum("ab,aic,bid->cd", E, c, c)
    return float(math.sqrt(max(E[0, 0], 0.0)))


# --------------------------------------------------------------------------------------
# closed-form structured trains (§4)
# --------------------------------------------------------------------------------------

def _xq(bases, a, h, q):
    """Quantized coordinate x_q = h * c_q * i_q; h = grid spacing."""
    c = digit_factors(bases)
    return h * c[q] * np.arange(bases[q], dtype=np.float64)


def exp_train(bases, a, h, v, x0) -> Train:
    """e^{v(x-x0)} as a rank-1 train, PAPER.md:335-344 (Eq. exp_dec)."""
    cores = []
    for q in range(len(bases)):
        val = np.exp(v * _xq(bases, a, h, q))
        if q == 0:
            val = val * math.exp(v * (a - x0))
        cores.append(val.reshape(1, -1, 1))
    return Train(cores, "mps")


def cos_train(bases, a, h, v, x0) -> Train:
    """cos(v(x-x0)) as a real rank-2 train, PAPER.md:401-430 (re-gauged rotation cores)."""
    n = len(bases)
    if n < 2:
        raise ValueError("cos_train needs at least two cores")
    cores = []
    for q in range(n):
        th = v * _xq(bases, a, h, q) + (v / n) * (a - x0)  # x~_q
        c, s = np.cos(th), np.sin(th)
        if q == 0:
            core = np.zeros((1, bases[q], 2))
            core[0, :, 0] = 0.5 * (c + s)
            core[0, :, 1] = 0.5 * (c - s)
        elif q == n - 1:
            core = np.zeros((2, bases[q], 1))
            core[0, :, 0] = c - s
            core[1, :, 0] = s + c
        else:
            core = np.zeros((2, bases[q], 2))
            core[0, :, 0] = c
            core[0, :, 1] = -s
            core[1, :, 0] = s
            core[1, :, 1] = c
        cores.append(core)
    return Train(cores, "mps")


def sin_train(bases, a, h, v, x0) -> Train:
    """sin(v(x-x0)) = cos(v(x - x0 - pi/(2v)))."""
    return cos_train(bases, a, h, v, x0 + math.pi / (2.0 * v))


def poly_train(bases, a, h, coeffs, x0) -> Train:
    """sum_t coeffs[t] (x-x0)^t as a rank-(p+1) train.

    The middle core is the lower-triangular reading C_q[s,t] = C(s,t) x~_q^{s-t}, t<=s
    (the printed formula PAPER.md:461-464 is transposed; SURVEY.md c-A23, A4)."""
    n = len(bases)
    p = len(coeffs) - 1
    cores = []
    for q in range(n):
        xt = _xq(bases, a, h, q) + (a - x0) / n  # x~_q
        d = bases[q]
        if q == 0:
            core = np.zeros((1, d, p + 1))
            for t in range(p + 1):
                core[0, :, t] = sum(coeffs[s] * math.comb(s, t) * xt ** (s - t) for s in range(t, p + 1))
        elif q == n - 1:
            core = np.zeros((p + 1, d, 1))
            for s in range(p + 1):
                core[s, :, 0] = xt ** s
        else:
            core = np.zeros((p + 1, d, p + 1))
            for s in range(p + 1):
                for t in range(s + 1):
                    core[s, :, t] = math.comb(s, t) * xt ** (s - t)
        cores.append(core)
    return Train(cores, "mps")


def mps_block_sum(a: Train, b: Train) -> Train:
    """Exact sum by block cores; used only to assemble inputs."""
    L = a.L
    cores = []
    for q in range(L):
        A, B = a.cores[q], b.cores[q]
        legs = A.shape[1:-1]
        if L == 1:
            cores.append(A + B)
            continue
        if q == 0:
            C = np.concatenate([A, B], axis=-1)
        elif q == L - 1:
            C = np.concatenate([A, B], axis=0)
        else:
            C = np.zeros((A.shape[0] + B.shape[0],) + legs + (A.shape[-1] + B.shape[-1],))
            C[: A.shape[0], ..., : A.shape[-1]] = A
            C[A.shape[0]:, ..., A.shape[-1]:] = B
        cores.append(C)
    return Train(cores, a.kind, a.leg_dim)


def scale_train(t: Train, s: float) -> Train:
    cores = [c.copy() for c in t.cores]
    cores[0] = cores[0] * s
    return Train(cores, t.kind, t.leg_dim)


# ----- shift matrices -----------------------------------------------

def _Qb(b: int, d: int) -> np.ndarray:
    """Q^b_d(i,j) = [i - j = d]; zero when d >= b."""
    M = np.zeros((b, b))
    if 0 <= d < b:
        for j in range(b - d):
            M[j + d, j] = 1.0
    return M


def _Rb(b: int, d: int) -> np.ndarray:
    """R^b_d = (Q^b_{b-d})^T."""
    return _Qb(b, b - d).T


def shift_train(bases: Sequence[int], d: int, select=(1.0, 0.0)) -> Train:
    """Q^N_d (select (1,0)), R^N_d (select (0,1)) or the circular shift (select (1,1)),
    from the rank-product factorization PAPER.md:514-529 with standard mixed-radix
    digits of d (SURVEY.md c-A24)."""
    n = len(bases)
    c = digit_factors(bases)
    N = math.prod(bases)
    if not (0 <= d <= N):
        raise ValueError("shift out of range")
    dig = []
    rem = d
    for q in range(n):
        dig.append(rem // c[q])
        rem -= dig[-1] * c[q]
    cores = []
    for q in range(n):
        b, dq = bases[q], dig[q]
        if q == n - 1:
            core = np.zeros((2, b, b, 1))
            core[0, :, :, 0] = _Qb(b, dq)
            core[1, :, :, 0] = _Rb(b, dq)
        else:
            core = np.zeros((2, b, b, 2))
            core[0, :, :, 0] = _Qb(b, dq)
            core[0, :, :, 1] = _Qb(b, dq + 1)
            core[1, :, :, 0] = _Rb(b, dq)
            core[1, :, :, 1] = _Rb(b, dq + 1)
        cores.append(core)
    sel = np.asarray(select, dtype=np.float64).reshape(1, 2)
    cores[0] = np.einsum("xa,aijb->xijb", sel, cores[0])
    return Train(cores, "mpo")


def mpo_transpose(t: Train) -> Train:
    return Train([np.ascontiguousarray(c.transpose(0, 2, 1, 3)) for c in t.cores], "mpo", t.leg_dim)


def stencil_rank8(bases: Sequence[int], weights=(1.0, -4.0, 6.0, -4.0, 1.0)) -> Train:
    """Banded shift-sum operator sum_{s=-2..2} w_s * shift_s, non-circular, as the exact
    rank-8 block sum of four rank-2 shift trains (SURVEY.md c-A20, A3):
    {Q_1 with last core -4 Q_1 + 6 Q_0 ; Q_2 ; -4 Q_1^T ; Q_2^T}."""
    w_m2, w_m1, w_0, w_p1, w_p2 = weights
    q1 = shift_train(bases, 1)
    q0 = shift_train(bases, 0)
    # Q_1 and Q_0 share every core but the last (digits of 1 = (0..0,1))
    last = w_p1 * q1.cores[-1] + w_0 * q0.cores[-1]
    a = Train(q1.cores[:-1] + [last], "mpo")
    q2 = scale_train(shift_train(bases, 2), w_p2)
    bt = scale_train(mpo_transpose(shift_train(bases, 1)), w_m1)
    ct = scale_train(mpo_transpose(shift_train(bases, 2)), w_m2)
    return mps_block_sum(mps_block_sum(mps_block_sum(a, q2), bt), ct)


def periodic_laplacian_1d(L: int) -> Train:
    """Periodic second-difference [1,-2,1] on N = 2^L (no 1/h^2), exact rank 3.

    Closed-form automaton over binary digits read from the least significant
    core: bond states {eq, carry, borrow} for j - i in {0,+1,-1} (mod N); circular
    wrap = sum over all three states at the most significant end (the (1,1)
    selection of PAPER.md:529 generalised).  Pinned against the dense stencil."""
    EQ, CA, BO = 0, 1, 2
    cores = []
    for q in range(L):
        last = (q == L - 1)
        core = np.zeros((3, 2, 2, 1 if last else 3))
        if last:
            # suffix empty: -2*[j=i] + [j=i+1] + [j=i-1]
            for i in range(2):
                core[EQ, i, i, 0] += -2.0
            core[EQ, 0, 1, 0] += 1.0   # j = i+1, no carry
            core[CA, 1, 0, 0] += 1.0   # j = i+1 with carry
            core[EQ, 1, 0, 0] += 1.0   # j = i-1, no borrow
            core[BO, 0, 1, 0] += 1.0   # j = i-1 with borrow
        else:
            for i in range(2):
                core[EQ, i, i, EQ] = 1.0
            core[EQ, 0, 1, CA] = 1.0   # need +1: i=0 -> j=1, done
            core[CA, 1, 0, CA] = 1.0   # i=1 -> j=0, carry on
            core[EQ, 1, 0, BO] = 1.0   # need -1: i=1 -> j=0, done
            core[BO, 0, 1, BO] = 1.0   # i=0 -> j=1, borrow on
        cores.append(core)
    cores[0] = cores[0].sum(axis=0, keepdims=True)  # circular: all states allowed at the top
    return Train(cores, "mpo")


def identity_mpo(dims: Sequence[int]) -> Train:
    return Train([np.eye(d).reshape(1, d, d, 1).copy() for d in dims], "mpo")


def interleave_mpo(t: Train, axis: int, n_axes: int, other_dims: Sequence[int]) -> Train:
    """Place a 1D MPO on every ``n_axes``-th site starting at ``axis`` (alternating
    digit layout x1,y1,x2,y2,..., SURVEY.md c-A19); pass-through cores
    delta_ij * delta_ww' on the other axes' sites."""
    cores = []
    L1 = t.L
    for q in range(L1):
        for ax in range(n_axes):
            if ax == axis:
                cores.append(t.cores[q])
            else:
                w = t.cores[q].shape[0] if ax < axis else t.cores[q].shape[-1]
                d = other_dims[q]
                core = np.einsum("ab,ij->aijb", np.eye(w), np.eye(d))
                cores.append(core)
    return Train(cores, "mpo")


def laplacian_2d_alternating(Lx: int) -> Train:
    """Delta_x (x) I + I (x) Delta_y, periodic, on the alternating layout x1,y1,...,x_n,y_n
    (SURVEY.md c-A19); block sum of the two interleaved rank-3 operators -> bonds <= 6."""
    l1 = periodic_laplacian_1d(Lx)
    ax = interleave_mpo(l1, 0, 2, [2] * Lx)
    ay = interleave_mpo(l1, 1, 2, [2] * Lx)
    out = mps_block_sum(ax, ay)
    out.leg_dim = [q % 2 for q in range(2 * Lx)]
    return out


# --------------------------------------------------------------------------------------
# the five configs (BASELINE.json configs[0..4])
# --------------------------------------------------------------------------------------

@dataclass
class Problem:
    name: str
    kind: str                  # "matvec" | "hadamard" | "truncate"
    op: Optional[Train]
    x: Train
    eps: float
    max_rank: int
    meta: dict = field(default_factory=dict)


def cfg1(L: int = 10) -> Problem:
    """configs[0]: sin(2 pi x) + x^2 on x_i = i/2^L (SURVEY.md c-A16), periodic Laplacian."""
    bases = [2] * L
    h = 1.0 / 2 ** L
    s = sin_train(bases, 0.0, h, 2.0 * math.pi, 0.0)
    p = poly_train(bases, 0.0, h, [0.0, 0.0, 1.0], 0.0)
    x = mps_block_sum(s, p)
    op = periodic_laplacian_1d(L)
    return Problem("cfg1", "matvec", op, x, 1e-12, 16, {"L": L})


def cfg2(Lx: int = 12, R: int = 64, max_rank: int = 128, eps: float = 1e-10) -> Problem:
    """configs[1]: 2D alternating layout, random N(0,1) state at rank R normalised to 1,
    periodic 5-point Laplacian (SURVEY.md c-A15, c-A19)."""
    dims = [2] * (2 * Lx)
    x = random_mps(dims, R, rng_for(2, 0, 0), 1.0)
    x = scale_train(x, 1.0 / env_norm(x))
    x.leg_dim = [q % 2 for q in range(2 * Lx)]
    op = laplacian_2d_alternating(Lx)
    return Problem("cfg2", "matvec", op, x, eps, max_rank, {"Lx": Lx, "R": R})


def cfg3(L: int = 30, R: int = 256, max_rank: int = 256, eps: float = 1e-8) -> Problem:
    """configs[2]: Hadamard 'i,i->i' of two random QTTs with N(0,1/R) cores (c-A14)."""
    dims = [2] * L
    std = 1.0 / math.sqrt(R)
    a = random_mps(dims, R, rng_for(3, 0, 0), std)
    b = random_mps(dims, R, rng_for(3, 0, 1), std)
    return Problem("cfg3", "hadamard", a, b, eps, max_rank, {"L": L, "R": R})


def cfg4(bases: Sequence[int] = tuple([3] * 8 + [5] * 4), R: int = 512, max_rank: int = 512,
         eps: float = 1e-12) -> Problem:
    """configs[3]: mixed radix 3^8*5^4, random state rank R N(0,1/R), rank-8 stencil."""
    bases = list(bases)
    x = random_mps(bases, R, rng_for(4, 0, 0), 1.0 / math.sqrt(R))
    op = stencil_rank8(bases)
    return Problem("cfg4", "matvec", op, x, eps, max_rank, {"bases": bases, "R": R})


def cfg5_member(b: int, L: int = 40, R: int = 64, W: int = 4, max_rank: int = 64,
                eps: float = 1e-10) -> Problem:
    """configs[4] member b: state rank R N(0,1/R) [2602,5,b,0]; MPO rank W N(0,1/W) [2602,5,b,1]."""
    dims = [2] * L
    x = random_mps(dims, R, rng_for(5, b, 0), 1.0 / math.sqrt(R))
    op = random_mpo(dims, W, rng_for(5, b, 1), 1.0 / math.sqrt(W))
    return Problem("cfg5", "matvec", op, x, eps, max_rank, {"L": L, "R": R, "W": W, "member": b})


def cfg5_batch_arrays(members: Sequence[int], L: int = 40, R: int = 64, W: int = 4):
    """Batch-strided arrays for cfg5: per site q one array (B, r_q, 2, r_{q+1}) / (B, w, 2, 2, w')."""
    probs = [cfg5_member(b, L, R, W) for b in members]
    xs = [np.stack([p.x.cores[q] for p in probs]) for q in range(L)]
    ops = [np.stack([p.op.cores[q] for p in probs]) for q in range(L)]
    return probs, xs, ops


# ----------------------------------------------------------------------------- Fourier (f2)

def qft_trains(bases_i: Sequence[int]) -> List[Train]:
    """The n rank-b_q factors of the DFT matrix M(i, j) = v^(i j), v = exp(-2 pi i / N)
    (Eq. for T(i_q, j)).  i = sum_q c^i_q i_q (big-endian, bases_i),
    j = sum_r c^j_r j_r with the reversed bases, and site k carries the digit pair
    (i_k, j_{n-k+1}) -- both of base b_k -- as one leg of size b_k^2 (i slow, j fast).
    Factor q = sum_s delta(s, i_q) prod_r exp(-2 pi i s c^i_q c^j_r j_r / N): a rank-b_q
    train whose bond carries s (block-diagonal cores; ones to sum s at the ends).  The
    phases are reduced mod N in integers before cos/sin.  Complex128 cores."""
    b = [int(x) for x in bases_i]
    n = len(b)
    N = int(np.prod(b))
    ci = digit_factors(b)
    bj = b[::-1]
    cj = digit_factors(bj)
    trains = []
    for q in range(n):
        bq = b[q]
        cores = []
        for k in range(n):
            bk = b[k]
            r = n - 1 - k                       # site k carries j_r (0-based r), base bj[r] == bk
            core = np.zeros((bq, bk * bk, bq), dtype=np.complex128)
            for s in range(bq):
                for ik in range(bk):
                    if k == q and ik != s:
                        continue
                    for jr in range(bk):
                        e = (s * ci[q] * cj[r] * jr) % N
                        core[s, ik * bk + jr, s] = np.exp(-2j * np.pi * e / N)
            if k == 0:
                core = core.sum(axis=0, keepdims=True)
            if k == n - 1:
                core = core.sum(axis=2, keepdims=True)
            cores.append(core)
        trains.append(Train(cores))
    return trains


def qft_dense_order(bases_i: Sequence[int]):
    """(shape, permutation) turning the dense tensor of a QFT-layout train (axes
    (i_1, j_n, i_2, j_{n-1}, ...)) into the N x N matrix with rows i and columns j."""
    b = [int(x) for x in bases_i]
    n = len(b)
    shape = []
    for k in range(n):
        shape += [b[k], b[k]]
    perm = [2 * k for k in range(n)] + [2 * (n - 1 - r) + 1 for r in range(n)]
    return shape, perm
