"""Jacobi phase cycles (diagnostics build -DQTT_JAC_PROFILE=1): runs the cfg5 batch once
through libqtt_jprof.so and prints cycles per round of each jac_round phase (warp 0)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["QTT_LIB"] = os.path.join(ROOT, "paper_2602_20226_b200", "lib", sys.argv[1] if len(sys.argv) > 1 else "libqtt_jprof.so")
sys.path.insert(0, ROOT)
import torch
from paper_2602_20226_b200 import gen, qtt
probs, xs, ops = gen.cfg5_batch_arrays(list(range(148)))
xd, od = qtt.to_device(xs), qtt.to_device(ops, mpo=True)
plan = qtt.ZipupPlan("ij,j->i", od, xd, 1e-10, 64)
plan.run(od, xd); torch.cuda.synchronize()
lib = qtt.load_library()
buf = (ctypes.c_ulonglong * 4)()
lib.qtt_debug_jprof(buf, 1)
plan.run(od, xd); torch.cuda.synchronize()
lib.qtt_debug_jprof(buf, 1)
r = buf[3]
print({"rounds": r, "dots_reduce": buf[0] / r, "params": buf[1] / r, "rotation": buf[2] / r,
       "total": (buf[0] + buf[1] + buf[2]) / r})
