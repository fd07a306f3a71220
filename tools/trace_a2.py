"""Timeline of the experimental 2-CTA kernel (A2_TRACE build, pair 0): leader MMA and both CTAs' softmax."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2506_04648_b200 as F
import paper_2506_04648_b200._lib as L
grid, tile, win, H, d = (21, 45, 80), (3, 5, 16), (5, 5, 3), 40, 128
Lt = grid[0] * grid[1] * grid[2]
q, k, v = (torch.randn((Lt, H, d), device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
plan = F.FpsaPlan(grid, tile, win, H, d)
plan.quantize(q, k, v); plan.attention(out); torch.cuda.synchronize()
buf = (ctypes.c_longlong * (3 * 128 * 4))()
L.lib().fpsa_a2_trace(buf)
T = np.array(buf, dtype=np.int64).reshape(3, 128, 4)
t0 = T[0, 2, 0]
print("step | MMA: wait-start p_ready-ok pv-issued qk-issued | leader sm warp: wait S-ready comp-end arrived | peer sm warp: ...")
for j in range(2, 128):
    m = T[0, j] - t0; a = T[1, j] - t0; b = T[2, j] - t0
    print(f"{j:3d} | {m[0]:8d} {m[1]:8d} {m[2]:8d} {m[3]:8d} | {a[0]:8d} {a[1]:8d} {a[2]:8d} {a[3]:8d} | {b[0]:8d} {b[1]:8d} {b[2]:8d} {b[3]:8d}")
