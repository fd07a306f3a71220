"""Run the C2 attention once with the FPSA_TRACE build and print where the cycles go."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_04648_b200._lib as L
L.LIB_PATH = L.LIB_PATH.replace("libfpsa.so", os.environ.get("FPSA_TRACE_LIB", "libfpsa_trace.so"))
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
print(f"   of which S load (tcgen05.ld + wait::ld, full blocks) {t[4]/n:.0f} clk")
steps = n / 8
print(f"MMA per step: wait P {t[3]/steps:.0f} clk, wait K/V {t[7]/steps:.0f} clk")
print(f"redo items: {t[5]} of {plan.n_items}")

# timeline of CTA 0: per step, softmax warps (wait start, S ready, compute end, P arrived) and MMA
tl = (ctypes.c_longlong * (256 * 10 * 4))()
lib.fpsa_trace_timeline.argtypes = [ctypes.POINTER(ctypes.c_longlong)]
lib.fpsa_trace_timeline(tl)
import numpy as np
T = np.array(tl, dtype=np.int64).reshape(256, 10, 4)
t0 = T[0, 0, 0]
print("step | warp0: wait S-ready comp-end arrived | warp4: ... | MMA: p_ready-ok pv-issued qk-issued   (clk rel. to step 0)")
for j in range(2, 40):
    w0 = T[j, 0] - t0; w4 = T[j, 4] - t0; w1 = T[j, 1] - t0; m = T[j, 9] - t0
    print(f"{j:3d} | {w0[0]:7d} {w0[1]:7d} {w0[2]:7d} {w0[3]:7d} | {w4[1]:7d} {w4[2]:7d} {w4[3]:7d} | w1 {w1[1]:7d} {w1[3]:7d} | {m[1]:7d} {m[2]:7d} {m[3]:7d}")

print("hand-off per step (clk): last owner arrival -> MMA at p_ready wait (TL0) / p_ready ok (TL1) / PV+QK issued (TL2) / S(j+2) ready at its owner")
rows = []
for j in range(4, 120):
    own = range(0, 4) if j % 2 == 0 else range(4, 8)
    arr = max(T[j, w, 3] for w in own)
    if arr <= 0 or T[j, 9, 1] <= 0 or T[j + 2, own[0], 1] <= 0:
        continue
    rows.append((T[j, 9, 0] - arr, T[j, 9, 1] - arr, T[j, 9, 2] - T[j, 9, 1], T[j + 2, own[0], 1] - T[j, 9, 2]))
if rows:
    r = np.array(rows)
    print("  mean: MMA at wait %+.0f, p_ready ok %+.0f, issue %.0f, QK->S ready %.0f" % tuple(r.mean(0)))
print("per-warp compute+store time (S-ready -> arrived), steps 2..60 mean, by warp (SMSP = warp % 4):")
for w in range(8):
    d = [T[j, w, 3] - T[j, w, 1] for j in range(2, 60) if T[j, w, 3] > 0]
    print(f"  warp {w} (SMSP {w % 4}): {np.mean(d):7.0f} clk")
