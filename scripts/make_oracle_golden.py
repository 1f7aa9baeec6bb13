#!/usr/bin/env python
"""Write the oracle's full-size results used by the slow GPU parity tests (calls only oracle/
through tests/oracle_cache.py, with the seeded generators for the inputs):

  cfg3_f64  configs[2] Hadamard, L=30, rank 256, max rank 256, eps 1e-8, fp64 inputs
  cfg3_f32  the same draws rounded to binary32 (SURVEY.md §8(d) "fp32 inputs"), fp64 oracle

  python scripts/make_oracle_golden.py [cfg3_f64 cfg3_f32]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from paper_2602_20226_b200 import gen  # noqa: E402
from oracle_cache import oracle_result  # noqa: E402


def f32(cores):
    return [np.asarray(c, dtype=np.float32).astype(np.float64) for c in cores]


def inputs(name):
    p = gen.cfg3()
    if name == "cfg3_f64":
        return "hadamard", p.op.cores, p.x.cores, p.eps, p.max_rank
    if name == "cfg3_f32":
        return "hadamard", f32(p.op.cores), f32(p.x.cores), p.eps, p.max_rank
    raise SystemExit(f"unknown {name}")


if __name__ == "__main__":
    for name in sys.argv[1:] or ["cfg3_f64", "cfg3_f32"]:
        kind, op, x, eps, mr = inputs(name)
        r = oracle_result(name, kind, op, x, eps, mr)
        print(name, r["ranks"], r["norm"], flush=True)
