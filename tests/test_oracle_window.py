"""Oracle pins for the window-N zip-up ("the first N-cores
(1 <= N <= n) are contracted exactly"): N = 1 is the N = 1 zip-up, N = L is the exact
product followed by TT-SVD, truncation with N = 2 keeps the identity
||y - x||^2 = sum delta^2, and eps -> 0 gives the exact product."""
import numpy as np
import pytest

from paper_2602_20226_b200 import gen
from oracle import tt
from oracle.zipup import zipup, zipup_window

DIMS = [2, 3, 2, 2, 5, 2]


def _ops(seed):
    rng = np.random.default_rng(seed)
    x = gen.random_mps(DIMS, 6, rng).cores
    op = gen.random_mpo(DIMS, 3, rng, 0.5).cores
    a = gen.random_mps(DIMS, 4, rng).cores
    return x, op, a


@pytest.mark.parametrize("kind", ["matvec", "hadamard", "truncate"])
def test_window1_is_the_zipup(kind):
    x, op, a = _ops(1)
    o = {"matvec": op, "hadamard": a, "truncate": None}[kind]
    r1, rw = zipup(kind, o, x, 1e-2, 5), zipup_window(kind, o, x, 1e-2, 5, 1)
    assert r1["ranks"] == rw["ranks"]
    for c1, cw in zip(r1["cores"], rw["cores"]):
        np.testing.assert_allclose(c1, cw, atol=1e-14)


@pytest.mark.parametrize("kind", ["matvec", "hadamard"])
def test_window_L_is_exact_product_then_tt_svd(kind):
    x, op, a = _ops(2)
    o = op if kind == "matvec" else a
    exact = tt.exact_matvec(op, x) if kind == "matvec" else tt.exact_hadamard(a, x)
    dense = tt.full_legs(exact).reshape(-1)
    ref, d2 = tt.tt_svd(dense, DIMS, 1e-3, 0)
    got = zipup_window(kind, o, x, 1e-3, 0, len(DIMS))
    assert got["ranks"] == [1] + [c.shape[-1] for c in ref]
    np.testing.assert_allclose(got["delta2"], d2, rtol=1e-9, atol=1e-24)
    y, yr = tt.full_legs(got["cores"]).reshape(-1), tt.full_legs(ref).reshape(-1)
    assert np.linalg.norm(y - yr) <= 1e-12 * np.linalg.norm(yr)


def test_window2_truncation_error_identity():
    x, _, _ = _ops(3)
    r = zipup_window("truncate", None, x, 0.05, 3, 2)
    e = tt.full_legs(r["cores"]) - tt.full_legs(x)
    assert abs(np.sum(e * e) - sum(r["delta2"])) <= 1e-12 * np.sum(tt.full_legs(x) ** 2)


@pytest.mark.parametrize("kind", ["matvec", "hadamard"])
def test_window2_eps0_is_exact(kind):
    x, op, a = _ops(4)
    o = op if kind == "matvec" else a
    exact = tt.exact_matvec(op, x) if kind == "matvec" else tt.exact_hadamard(a, x)
    r = zipup_window(kind, o, x, 0.0, 0, 2)
    y, ye = tt.full_legs(r["cores"]), tt.full_legs(exact)
    assert np.linalg.norm(y - ye) <= 1e-12 * np.linalg.norm(ye)
    for q in range(1, len(DIMS)):                 # c-A35: never above the exact product's bond
        assert r["ranks"][q] <= exact[q].shape[0]
