#!/usr/bin/env python
"""Small zip-ups for compute-sanitizer (racecheck / synccheck / memcheck), SURVEY.md §4 T5:
  small   : a 16-member cfg5 batch through k_orth + k_sweep (task queue with acquire/release flags)
  large   : reduced cfg2 (m = 256) through the large-member path (k_qr_coop / k_jacobi_coop grid
            barriers, dataflow flags)
  window2 : a 4-member cfg5 batch with QTT_WINDOW2 (k_zipup<double>)
  var2    : two-site variational on 2 cfg5 members"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2602_20226_b200 import gen, qtt  # noqa: E402


def main(which):
    torch.cuda.set_device(0)
    if which in ("small", "window2", "var2"):
        n = {"small": 16, "window2": 4, "var2": 2}[which]
        probs, xs, ops = gen.cfg5_batch_arrays(list(range(n)))
        xd, od = qtt.to_device(xs), qtt.to_device(ops, mpo=True)
        if which == "var2":
            z = qtt.ZipupPlan("ij,j->i", od, xd, 1e-10, 8).run(od, xd)
            v = qtt.variational("ij,j->i", od, xd, z, 1, ncores=2, max_rank=16)
            torch.cuda.synchronize()
            assert int(v.status.item()) == 0
        else:
            flags = qtt.WINDOW2 if which == "window2" else 0
            r = qtt.ZipupPlan("ij,j->i", od, xd, 1e-10, 64, flags=flags).run(od, xd)
            torch.cuda.synchronize()
            assert int(r.status.item()) == 0
    elif which == "large":
        p = gen.cfg2(Lx=6, R=64, max_rank=128)
        xd, od = qtt.to_device(p.x.cores), qtt.to_device(p.op.cores, mpo=True)
        r = qtt.ZipupPlan("ij,j->i", od, xd, p.eps, p.max_rank).run(od, xd)
        torch.cuda.synchronize()
        assert int(r.status.item()) == 0
    print("ok", which, flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
