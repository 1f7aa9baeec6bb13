import os, sys, math
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from paper_2602_20226_b200 import gen, qtt
from oracle import tt
from test_gpu_large import _redundant_ones
L, R = 30, 256
ones = _redundant_ones(L, R)
a = gen.random_mps([2] * L, R, gen.rng_for(3, 0, 0), 1.0 / math.sqrt(R)).cores
dig = np.random.default_rng(9).integers(0, 2, size=(256, L))
for name, x in (("ones", ones), ("a", a)):
    xd = qtt.to_device(x)
    r = qtt.ZipupPlan("i->i", None, xd, 0.0, 0).run(None, xd)
    torch.cuda.synchronize()
    rk = r.ranks[0].cpu().tolist()
    y = qtt.member_cores(r.out, rk, 0)
    ye, xe = tt.evaluate(y, dig), tt.evaluate(x, dig)
    print(name, "status", int(r.status.item()), "max ratio", float(np.max(np.abs(ye / xe))), "min", float(np.min(np.abs(ye / xe))),
          "ranks", rk[:12], flush=True)
