"""Print dependent-chain latencies (cycles) of FP64 ops on this GPU and the raw error of the
f64 MUFU approximations (csrc/probe/lat.cu).  Diagnostics for kernel design only."""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2602_20226_b200", "lib", "libqttprobe.so"))
out = torch.zeros(16, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
for _ in range(2):
    lib.qtt_probe_latency(ctypes.c_void_p(out.data_ptr()), 4096, ctypes.c_void_p(s.cuda_stream))
torch.cuda.synchronize()
v = out.cpu().tolist()
print({"dfma": v[0], "shfl64": v[1], "rsqrt_approx": v[2], "rcp_approx": v[3], "lds64_chase": v[4], "dadd": v[5],
       "rsqrt_approx_max_rel_err": v[8], "rcp_approx_max_rel_err": v[9]})
out.zero_()
for _ in range(2):
    lib.qtt_probe_tput(ctypes.c_void_p(out.data_ptr()), 20000, 148, ctypes.c_void_p(s.cuda_stream))
torch.cuda.synchronize()
v = out.cpu().tolist()
print({"shfl32_cycles_per_instr_per_SM": v[0], "lds64_bcast_cycles_per_instr_per_SM": v[1]})
out.zero_()
lib.qtt_probe_rsqrt_err(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s.cuda_stream))
torch.cuda.synchronize()
print({"halley_rsqrt_max_rel_err": out[0].item()})
