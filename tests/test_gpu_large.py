"""GPU parity of the large-member path (site matrices with m > 128 rows: cooperative
Householder QR, cooperative block Jacobi, strided GEMMs) against the oracle, on
configs[1..3] shapes (reduced and full where the oracle finishes in reasonable time)."""
import math

import numpy as np
import pytest

from paper_2602_20226_b200 import gen
from parity import compare

from test_gpu_zipup import check, member, run_gpu

pytestmark = pytest.mark.gpu


def test_large_truncate_random(lib):
    x = gen.random_mps([3] * 7, 300, np.random.default_rng(2)).cores      # bonds up to 243 -> m up to 729
    check(lib, "truncate", None, x, 1e-10, 0, dense=True)


def test_large_cfg2_reduced_m256(lib):
    p = gen.cfg2(Lx=6, R=64, max_rank=128)
    check(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank)


def test_large_cfg4_reduced_mixed_radix(lib):
    p = gen.cfg4(bases=(3, 3, 3, 5, 5), R=64, max_rank=64)
    check(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank)


def test_large_cfg3_reduced_hadamard(lib):
    p = gen.cfg3(L=14, R=128, max_rank=128)
    check(lib, "hadamard", p.op.cores, p.x.cores, p.eps, p.max_rank, dense=True)


@pytest.mark.slow
def test_cfg2_full(lib):
    """configs[1] at full size: L=24, rank 64, max rank 128, eps 1e-10 (2^24 entries: dense ok)."""
    p = gen.cfg2()
    check(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank, dense=False)


@pytest.mark.slow
def test_cfg4_full(lib):
    """configs[3] at full size: 3^8*5^4 mixed radix, rank 512, rank-8 stencil, max rank 512."""
    p = gen.cfg4()
    check(lib, "matvec", p.op.cores, p.x.cores, p.eps, p.max_rank, dense=False)
