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
