"""Oracle pins for the variational refinement:
the distance never increases (|O - C|^2 = |O|^2 - |C_q|^2 at the centre), that identity
itself against the dense distance, an exact seed stays exact, and the last update is the
brute-force least-squares optimum of the centre core given the others (Eq. variational)."""
import numpy as np
import pytest

from paper_2602_20226_b200 import gen
from oracle import tt
from oracle.variational import variational
from oracle.zipup import zipup


def _problem(kind, seed=5):
    rng = np.random.default_rng(seed)
    dims = [2] * 9
    x = gen.random_mps(dims, 8, rng).cores
    op = {"matvec": gen.random_mpo(dims, 3, rng, 0.5).cores, "hadamard": gen.random_mps(dims, 3, rng).cores,
          "truncate": None}[kind]
    ex = {"matvec": lambda: tt.exact_matvec(op, x), "hadamard": lambda: tt.exact_hadamard(op, x),
          "truncate": lambda: x}[kind]()
    return op, x, ex


@pytest.mark.parametrize("kind", ["matvec", "hadamard", "truncate"])
def test_monotone_and_distance_identity(kind):
    op, x, ex = _problem(kind)
    z = zipup(kind, op, x, 0.2, 5)
    v = variational(kind, op, x, z["cores"], 3)
    n = v["center_norm2"]
    nO = tt.inner(ex, ex)
    assert all(n[i + 1] >= n[i] - 1e-12 * nO for i in range(len(n) - 1))
    d2 = tt.diff_norm(v["cores"], ex) ** 2
    assert abs(d2 - (nO - n[-1])) <= 1e-9 * nO
    assert d2 <= tt.diff_norm(z["cores"], ex) ** 2 * (1 + 1e-12)


def test_exact_seed_stays_exact():
    op, x, ex = _problem("matvec", 6)
    z = zipup("matvec", op, x, 0.0, 0)
    v = variational("matvec", op, x, z["cores"], 1)
    assert tt.diff_norm(v["cores"], ex) <= 1e-10 * tt.qr_norm(ex)


def test_last_update_is_the_least_squares_optimum():
    """After the final left sweep the centre is C_0 and C_1.. are right-orthonormal: C_0 must
    equal the projection of the exact result onto their span (brute force, dense)."""
    op, x, ex = _problem("matvec", 7)
    z = zipup("matvec", op, x, 0.3, 4)
    v = variational("matvec", op, x, z["cores"], 2)
    C = v["cores"]
    # dense right basis B[a, rest] of C_1..C_{L-1}
    acc = C[-1].reshape(C[-1].shape[0], -1)
    for c in reversed(C[1:-1]):
        acc = (c.reshape(-1, c.shape[-1]) @ acc).reshape(c.shape[0], -1)
    B = acc
    np.testing.assert_allclose(B @ B.T, np.eye(B.shape[0]), atol=1e-12)
    O = tt.full_legs(ex).reshape(C[0].shape[1], -1)
    C0 = (O @ B.T).reshape(C[0].shape)
    np.testing.assert_allclose(C[0], C0, atol=1e-10 * np.abs(C0).max())


# ------------------------------------------------------------------ two-site (ncores = 2)
# PAPER.md:300 (multi-core super-cores, rank control), PAPER.md:794 (ncores=2), reading c-A37.

def _dense_dist2(C, ex):
    return float(np.sum((tt.to_dense_vector(C) - tt.to_dense_vector(ex)) ** 2))


@pytest.mark.parametrize("kind", ["matvec", "hadamard", "truncate"])
def test_two_site_monotone_and_identity(kind):
    """cutoff 0 and max_rank at least the seed's ranks: every split's feasible set contains the
    current state, so |S_k|^2 never decreases; and |O - C|^2 = |O|^2 - |S_k|^2 (dense)."""
    op, x, ex = _problem(kind, 9)
    z = zipup(kind, op, x, 0.2, 4)
    v = variational(kind, op, x, z["cores"], 2, ncores=2, eps=0.0, max_rank=6)
    n = v["center_norm2"]
    nO = float(np.sum(tt.to_dense_vector(ex) ** 2))
    assert len(n) == 2 * 2 * (len(x) - 1)
    assert all(n[i + 1] >= n[i] - 1e-12 * nO for i in range(len(n) - 1))
    d2 = _dense_dist2(v["cores"], ex)
    assert abs(d2 - (nO - n[-1])) <= 1e-10 * nO
    assert d2 <= _dense_dist2(z["cores"], ex) * (1 + 1e-12)
    assert max(v["ranks"]) <= 6


def test_two_site_grows_ranks_to_exact():
    """From a rank-1 seed, two-site sweeps with max_rank >= the exact ranks and cutoff 0 reach
    the exact product (dense), which single-site sweeps cannot (their ranks stay 1)."""
    rng = np.random.default_rng(31)
    dims = [2] * 6
    x = gen.random_mps(dims, 3, rng).cores
    op = gen.random_mpo(dims, 2, rng, 0.5).cores
    ex = tt.exact_matvec(op, x)
    seed = [np.ones((1, 2, 1)) for _ in dims]
    v2 = variational("matvec", op, x, seed, 3, ncores=2, eps=0.0, max_rank=64)
    yo = tt.to_dense_vector(ex)
    assert np.linalg.norm(tt.to_dense_vector(v2["cores"]) - yo) <= 1e-10 * np.linalg.norm(yo)
    v1 = variational("matvec", op, x, seed, 3)
    assert max(v1["ranks"]) == 1
    assert np.linalg.norm(tt.to_dense_vector(v1["cores"]) - yo) >= 1e-2 * np.linalg.norm(yo)


def test_two_site_split_is_truncated_svd_of_the_optimum():
    """One pair update with max_rank unbounded and cutoff 0 is the least-squares optimum of the
    super-core given the other (orthonormal) cores; with max_rank k the kept part is its best
    rank-k approximation (Eckart-Young): checked by brute force on the dense result."""
    op, x, ex = _problem("matvec", 10)
    z = zipup("matvec", op, x, 0.3, 3)
    v = variational("matvec", op, x, z["cores"], 1, ncores=2, eps=0.0, max_rank=3)
    C = v["cores"]                       # centre at site 0: C_1.. right-orthonormal
    acc = C[-1].reshape(C[-1].shape[0], -1)
    for c in reversed(C[2:-1]):
        acc = (c.reshape(-1, c.shape[-1]) @ acc).reshape(c.shape[0], -1)
    B = acc                              # right basis of sites 2.. (a, rest)
    np.testing.assert_allclose(B @ B.T, np.eye(B.shape[0]), atol=1e-12)
    O = tt.full_legs(ex).reshape(2 * 2, -1)   # rows (i0, i1)
    S_opt = (O @ B.T)                          # (i0 i1) x a, the optimum super-core
    M = S_opt.reshape(2, 2 * B.shape[0])       # (c=1 * d0) x (d1 * a)
    s = np.linalg.svd(M, compute_uv=False)
    k = min(3, s.size)
    got = np.einsum("cia,ajb->cijb", C[0], C[1]).reshape(2, -1)
    assert abs(np.sum(got ** 2) - np.sum(s[:k] ** 2)) <= 1e-10 * np.sum(s ** 2)
    # and the kept part is the best rank-k approximation
    U, s2, Vh = np.linalg.svd(M, full_matrices=False)
    best = (U[:, :k] * s2[:k]) @ Vh[:k]
    np.testing.assert_allclose(got, best, atol=1e-10 * np.abs(best).max())


def test_two_site_truncation_rule_controls_ranks():
    """cutoff > 0: ranks follow the SPEC.md:299 rule on each super-core; a larger cutoff never
    gives larger ranks (same seed)."""
    op, x, ex = _problem("matvec", 11)
    z = zipup("matvec", op, x, 0.0, 0)
    lo = variational("matvec", op, x, z["cores"], 1, ncores=2, eps=1e-1, max_rank=0)
    hi = variational("matvec", op, x, z["cores"], 1, ncores=2, eps=1e-6, max_rank=0)
    assert all(a <= b for a, b in zip(lo["ranks"], hi["ranks"]))
    assert sum(lo["ranks"]) < sum(hi["ranks"])
    nO = float(np.sum(tt.to_dense_vector(ex) ** 2))
    assert _dense_dist2(hi["cores"], ex) <= 1e-8 * nO
