"""QR phase cycles of the small path (diagnostics build -DQTT_JAC_PROFILE=1): cfg5 batch of 148
members once through the given library; prints cycles per qr_of_TH call of each phase."""
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
buf = (ctypes.c_ulonglong * 24)()
lib.qtt_debug_jprof(buf, 1)
plan.run(od, xd); torch.cuda.synchronize()
lib.qtt_debug_jprof(buf, 1)
n = max(buf[10], 1)
r = max(buf[3], 1)
print({"qr_calls": n, "qr_total": buf[11] / n, "staging": buf[4] / n, "w0_small_trailing": buf[6] / n,
       "w0_panel": buf[5] / n, "w0_wait": buf[8] / n, "w1_big_trailing": buf[7] / n, "w1_wait": buf[9] / n})
no = max(buf[15], 1)
print({"orth_sites_128x64": buf[15], "factor": buf[12] / no, "form_q": buf[13] / no, "absorb_gemm": buf[14] / no,
       "  of which Q^T out": buf[20] / no, "prev staging": buf[21] / no})
nc = max(buf[18], 1)
print({"a2_warp_tiles": buf[18], "a2_total_per_warp": buf[16] / nc, "a2_dmma_per_warp": buf[17] / nc, "a2_staging_per_site": buf[19] / max(buf[18] / 8, 1)})
print({"jac_rounds": r, "dots_reduce": buf[0] / r, "params": buf[1] / r, "rotation": buf[2] / r})
