"""GPU parity of the window-2 zip-up (QTT_WINDOW2) against the oracle's
zipup_window(..., 2), by the tests/parity.py protocol: random MPO / Hadamard / truncation
(mixed radix included), a cfg5 member (L = 40, rank 64: 128 x 512 super-cores), a complex
Hadamard, and a batch; plus accuracy against the N = 1 zip-up on the same input."""
import math

import numpy as np
import pytest

from paper_2602_20226_b200 import gen
from parity import compare

pytestmark = pytest.mark.gpu


def run_w2(lib, subs, op, x, eps, max_rank, mpo=False, dtype=np.float64):
    import torch
    xd = lib.to_device(x, dtype=dtype)
    od = None if op is None else lib.to_device(op, mpo=mpo, dtype=dtype)
    plan = lib.ZipupPlan(subs, od, xd, eps, max_rank, flags=lib.WINDOW2, sigma_stride=512)
    res = plan.run(od, xd)
    torch.cuda.synchronize()
    assert int(res.status.item()) == 0, int(res.status.item())
    return res


def check_w2(lib, kind, op, x, eps, max_rank, b=0, dense=True, res=None, dtype=np.float64):
    subs = {"matvec": "ij,j->i", "hadamard": "i,i->i", "truncate": "i->i"}[kind]
    if res is None:
        res = run_w2(lib, subs, op, x, eps, max_rank, mpo=(kind == "matvec"), dtype=dtype)
    ranks = res.ranks[b].cpu().tolist()
    cores = lib.member_cores(res.out, ranks, b)
    return compare(kind, op, x, eps, max_rank, cores, ranks, res.sigma[b].cpu().numpy(), res.delta2[b].cpu().numpy(),
                   float(res.norm2[b].item()), dense=dense, window=2)


@pytest.mark.parametrize("dims,R,W,mr,eps", [([2] * 10, 12, 3, 16, 1e-10), ([2, 3, 2, 5, 3, 2, 2], 9, 4, 0, 0.0),
                                             ([2] * 12, 16, 3, 8, 1e-6)])
def test_window2_matvec(lib, dims, R, W, mr, eps):
    x = gen.random_mps(dims, R, np.random.default_rng(len(dims) * 3 + R)).cores
    op = gen.random_mpo(dims, W, np.random.default_rng(len(dims) * 5 + W), 0.5).cores
    check_w2(lib, "matvec", op, x, eps, mr)


def test_window2_hadamard_and_truncate(lib):
    a = gen.random_mps([2] * 11, 8, np.random.default_rng(61), 1 / math.sqrt(8)).cores
    b = gen.random_mps([2] * 11, 8, np.random.default_rng(62), 1 / math.sqrt(8)).cores
    check_w2(lib, "hadamard", a, b, 1e-8, 20)
    check_w2(lib, "truncate", None, gen.random_mps([3] * 7, 20, np.random.default_rng(63)).cores, 1e-3, 0)


def test_window2_complex_hadamard(lib):
    rng = np.random.default_rng(64)
    a = [c + 1j * rng.standard_normal(c.shape) for c in gen.random_mps([2] * 9, 6, rng).cores]
    b = [c + 1j * rng.standard_normal(c.shape) for c in gen.random_mps([2] * 9, 6, rng).cores]
    check_w2(lib, "hadamard", a, b, 1e-10, 12, dtype=np.complex128)


def test_window2_cfg5_members_and_accuracy(lib):
    """configs[4] shapes with QTT_WINDOW2 on a 3-member batch; window 2 is at least as
    accurate as window 1 on these members (its splits see one more site)."""
    import torch
    from oracle import tt
    members = [0, 7, 300]
    probs, xs, ops = gen.cfg5_batch_arrays(members)
    xd, od = lib.to_device(xs), lib.to_device(ops, mpo=True)
    plan = lib.ZipupPlan("ij,j->i", od, xd, 1e-10, 64, flags=lib.WINDOW2, sigma_stride=512)
    res = plan.run(od, xd)
    torch.cuda.synchronize()
    assert int(res.status.item()) == 0
    p1 = lib.ZipupPlan("ij,j->i", od, xd, 1e-10, 64)
    r1 = p1.run(od, xd)
    torch.cuda.synchronize()
    for i, p in enumerate(probs):
        out = check_w2(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank, b=i, dense=False, res=res)
        y2 = lib.member_cores(res.out, res.ranks[i].cpu().tolist(), i)
        y1 = lib.member_cores(r1.out, r1.ranks[i].cpu().tolist(), i)
        ex = tt.exact_matvec(p.op.cores, p.x.cores)
        e2, e1 = tt.diff_norm(y2, ex), tt.diff_norm(y1, ex)
        assert e2 <= 1.05 * e1 + 1e-12 * tt.qr_norm(ex), (e2, e1)


def test_window2_wide_bonds(lib):
    """Bonds of 128 (x) exceed k_orth's shared-memory staging budget: the real window-2 path must
    fall back to its global-memory a1 instead of overrunning shared memory."""
    x = gen.random_mps([2] * 14, 128, np.random.default_rng(71), 1 / math.sqrt(128)).cores
    op = gen.random_mpo([2] * 14, 3, np.random.default_rng(72), 0.5).cores
    assert max(c.shape[0] for c in x) == 128
    check_w2(lib, "matvec", op, x, 1e-8, 40, dense=False)
    check_w2(lib, "truncate", None, x, 1e-3, 24, dense=False)
