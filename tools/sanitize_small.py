"""Small FP8 + passthrough runs for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_04648_b200 as fpsa

grid, tile, win, H, d = (6, 10, 32), (3, 5, 16), (3, 3, 3), 2, 128
L = grid[0] * grid[1] * grid[2]
g = torch.Generator(device="cuda").manual_seed(3)
q, k, v = (torch.randn((L, H, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
out = fpsa.FpsaPlan(grid, tile, win, H, d)(q, k, v, "lhd")
redo = fpsa.FpsaPlan(grid, tile, win, H, d, tau=0.0)  # forces the exact-mode launch
redo(q, k, v, "lhd")
norm = fpsa.FpsaPlan(grid, tile, win, H, d, p_mode="normalized")  # three-pass normalised-P launch
nout = torch.empty((L, H, d), dtype=torch.float32, device="cuda")
norm.quantize(q, k, v, "lhd")
norm.attention(nout, "lhd")
ties = (torch.randint(-255, 256, (L, H, d), generator=g, device="cuda").float() / 64.0)
ties[0::240, :, 0] = 4.25
ties = ties.to(torch.bfloat16)
fpsa.FpsaPlan(grid, tile, win, H, d).quantize(ties, ties, ties, "lhd")  # tie-rich tiles: the tie table
pt = fpsa.PassthroughPlan(grid, tile, win, H, d)(q, k, v, "lhd", out_dtype=torch.float32)
fid = fpsa.device_fidelity(pt, out.float(), "lhd")
torch.cuda.synchronize()
print("ok", redo.redo_count(), fid[0])
