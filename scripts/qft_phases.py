# per-phase clocks of the complex zip-up over one 2^13 Fourier chain (rank 16)
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_20226_b200 import gen, qtt
T = [t.cores for t in gen.qft_trains([2] * 13)]
dev = [qtt.to_device(t, dtype=np.complex128) for t in T]
for rep in range(2):
    y = dev[0]; tot = np.zeros(5); keep = []
    for q in range(1, 13):
        plan = qtt.ZipupPlan("i,i->i", dev[q], y, 0.0, 16, cycles=True, sweeps=True)
        res = plan.run(dev[q], y)
        c = res.cycles[0].cpu().numpy().astype(float)
        tot[4] += c[0, 3]; c[0, 3] = 0
        tot[:4] += c.sum(axis=0)
        ranks = res.ranks[0].cpu().tolist(); y = qtt.member_view(res.out, ranks, 0); keep.append(plan)
    print("Mcycles: a2 %.2f a3 %.2f a4 %.2f a5a6 %.2f a1 %.2f" % tuple(tot / 1e6))
