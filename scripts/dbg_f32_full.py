"""Diagnostics of the fp32 variant at full cfg3 size vs the cached fp64 oracle: per-site sigma
error (relative to s_1), delta2 error, rel_fro."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from paper_2602_20226_b200 import gen, qtt
from oracle import tt
from oracle_cache import oracle_result
f32 = lambda cs: [np.asarray(c, dtype=np.float32).astype(np.float64) for c in cs]
p = gen.cfg3()
op, x = f32(p.op.cores), f32(p.x.cores)
ref = oracle_result("cfg3_f32", "hadamard", op, x, p.eps, p.max_rank)
for dt in (np.float32, np.float64):
    xd, od = qtt.to_device(x, dtype=dt), qtt.to_device(op, dtype=dt)
    r = qtt.ZipupPlan("i,i->i", od, xd, p.eps, p.max_rank, sigma_stride=512).run(od, xd)
    torch.cuda.synchronize()
    rk = r.ranks[0].cpu().tolist()
    sg = r.sigma[0].cpu().numpy()
    errs = []
    for q in range(len(x) - 1):
        so = ref["sigmas"][q]; k = ref["ranks"][q + 1]; n = min(so.size, k + 4)
        errs.append(float(np.max(np.abs(sg[q][:n] - so[:n])) / so[0]))
    y = qtt.member_cores(r.out, rk, 0)
    rel = tt.diff_norm(y, ref["cores"]) / tt.qr_norm(ref["cores"])
    print(dt.__name__, "ranks_equal", rk == ref["ranks"], "rel_fro %.3e" % rel)
    print("  sigma err per site:", " ".join("%.1e" % e for e in errs))
