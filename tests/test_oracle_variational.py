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
