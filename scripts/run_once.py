#!/usr/bin/env python
"""One zip-up of a BASELINE config through the C-ABI (for ncu captures): run_once.py cfg3 [f32]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2602_20226_b200 import gen, qtt
w = sys.argv[1]
dt = np.float32 if len(sys.argv) > 2 and sys.argv[2] == "f32" else np.float64
p = {"cfg2": gen.cfg2, "cfg3": gen.cfg3, "cfg4": gen.cfg4}[w]()
subs = {"matvec": "ij,j->i", "hadamard": "i,i->i"}[p.kind]
xd = qtt.to_device(p.x.cores, dtype=dt)
od = qtt.to_device(p.op.cores, mpo=(p.kind == "matvec"), dtype=dt)
plan = qtt.ZipupPlan(subs, od, xd, p.eps, p.max_rank)
r = plan.run(od, xd)
torch.cuda.synchronize()
print(w, "status", int(r.status.item()), "ranks", r.ranks[0].tolist())
