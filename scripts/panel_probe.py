"""Cycles of the small path's QR pieces in isolation (probe/panel.cu): one 8-column panel
(all 16 panels of a 128-column block, other warps idle) and a whole qr_of_TH (128 x 256)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import torch
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2602_20226_b200", "lib", sys.argv[1] if len(sys.argv) > 1 else "libqttprobe.so"))
g = torch.Generator().manual_seed(5)
T = torch.randn(128, 256, generator=g, dtype=torch.float64).cuda()
out = (ctypes.c_longlong * 1)()
for mode, name in ((0, "16 panels (one warp)"), (1, "qr_of_TH 128x256")):
    lib.qtt_probe_panel(ctypes.c_void_p(T.data_ptr()), out, mode, 20)
    lib.qtt_probe_panel(ctypes.c_void_p(T.data_ptr()), out, mode, 20)
    print(name, out[0], "cycles")
c0 = torch.randn(64, 128, generator=g, dtype=torch.float64).cuda()
p0 = torch.randn(128, 64, generator=g, dtype=torch.float64).cuda()
c1, p1 = torch.empty_like(c0), torch.empty_like(p0)
for _ in range(2):
    lib.qtt_probe_orth(ctypes.c_void_p(c0.data_ptr()), ctypes.c_void_p(p0.data_ptr()), ctypes.c_void_p(c1.data_ptr()),
                       ctypes.c_void_p(p1.data_ptr()), out, 10)
print("a1 site 64x128 (orth_site_reg<4,8>)", out[0], "cycles")
# check: rows of the new core orthonormal, prev' core' == prev core
Q = c1.cpu(); print("  |Q Q^T - I| =", float((Q @ Q.T - torch.eye(64, dtype=torch.float64)).abs().max()),
                    " |P'Q' - P C| =", float((p1.cpu() @ Q - p0.cpu() @ c0.cpu()).abs().max()))
for _ in range(2):
    lib.qtt_probe_orthblk(ctypes.c_void_p(c0.data_ptr()), ctypes.c_void_p(p0.data_ptr()), ctypes.c_void_p(c1.data_ptr()),
                          ctypes.c_void_p(p1.data_ptr()), out, 10)
print("a1 site 64x128 (orth_site_blk)", out[0], "cycles")
Q = c1.cpu(); print("  |Q Q^T - I| =", float((Q @ Q.T - torch.eye(64, dtype=torch.float64)).abs().max()),
                    " |P'Q' - P C| =", float((p1.cpu() @ Q - p0.cpu() @ c0.cpu()).abs().max()))
tr = (ctypes.c_longlong * 128)()
lib.qtt_probe_blktrace(tr)
for st in range(8):
    o = tr[st * 8: st * 8 + 8]
    print(f"  step {st}: panel-warp small {o[0]:6d} panel {o[1]:6d} wait {o[2]:6d} | warp0 small {o[4]:6d} big {o[5]:6d} wait {o[6]:6d}")
lib.qtt_probe_blktrace(tr)
for w in range(8):
    o = tr[64 + w * 8: 64 + w * 8 + 4]
    print(f"  absorb warp {w}: Q^T out {o[0]:6d} staging {o[1]:6d} gemm+stores {o[2]:6d} final barrier {o[3]:6d}")
