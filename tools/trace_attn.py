"""Run the C2 attention once with the FPSA_TRACE build and print where the cycles go."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_04648_b200._lib as L
L.LIB_PATH = L.LIB_PATH.replace("libfpsa.so", "libfpsa_trace.so")
import torch
import paper_2506_04648_b200 as F
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
grid, tile, win, H = {"c2": ((21, 45, 80), (3, 5, 16), (5, 5, 3), 40), "c1": ((21, 30, 52), (3, 10, 4), (3, 3, 5), 12)}[cfg]
d = 128; Lt = grid[0] * grid[1] * grid[2]
q, k, v = (torch.randn((Lt, H, d), device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
plan = F.FpsaPlan(grid, tile, win, H, d)
plan.quantize(q, k, v); plan.attention(out); torch.cuda.synchronize()
lib = L.lib(); fn = lib.fpsa_trace_read; fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 8)(); fn(buf, 1)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); plan.attention(out); e.record(); torch.cuda.synchronize()
fn(buf, 1)
t = list(buf)
n_sm_warps = t[6]  # sum over softmax warps of n_kv
print(f"attention {s.elapsed_time(e):.3f} ms (traced build)")
n = max(1, t[6])  # softmax warp-steps
print(f"softmax per warp-step: loop {t[1]/n:.0f} clk, wait-for-S {t[0]/n:.0f}, first-pass compute {t[2]/n:.0f}, "
      f"rest (setup/store/arrive) {(t[1]-t[0]-t[2])/n:.0f}")
steps = n / 8
print(f"MMA per step: wait P {t[3]/steps:.0f} clk, wait K/V {t[7]/steps:.0f} clk")
print(f"redo items: {t[5]} of {plan.n_items}")
