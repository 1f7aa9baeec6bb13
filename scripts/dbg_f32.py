import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import math, numpy as np, torch
from paper_2602_20226_b200 import gen, qtt as lib
from test_gpu_large import _redundant_ones
def f32(c): return [np.asarray(x, dtype=np.float32).astype(np.float64) for x in c]
L, R = 30, 256
a = f32(gen.random_mps([2] * L, R, gen.rng_for(3, 0, 0), 1.0 / math.sqrt(R)).cores)
ones = f32(_redundant_ones(L, R))
for dt in (np.float64, np.float32):
    xd = lib.to_device(a, dtype=dt); od = lib.to_device(ones, dtype=dt)
    plan = lib.ZipupPlan("i,i->i", od, xd, 1e-8, 256, sigma_stride=512, sweeps=True)
    res = plan.run(od, xd); torch.cuda.synchronize()
    sig = res.sigma[0].cpu().numpy()
    print(lib.LIB_PATH[-16:], dt.__name__, "status", int(res.status.item()), "ranks", res.ranks[0].cpu().tolist()[5:12],
          "sweeps", res.sweeps[0].cpu().tolist()[5:12], "zero-sigma", [int((sig[q] == 0).sum()) for q in range(5, 12)], flush=True)
