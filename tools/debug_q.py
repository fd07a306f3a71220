import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O
import paper_2506_04648_b200 as F
grid, tile, win, H, d = (6, 10, 32), (3, 5, 16), (3, 3, 3), 1, 128
L = 1920; tv = 240
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn((L, H, d), generator=g, device="cuda").to(torch.bfloat16)
perm = O.tile_perm(grid, tile)
for dt in (torch.bfloat16, torch.float32):
    for nat in (True, False):
        xx = x.to(dt)
        if not nat:
            xx = xx[perm].contiguous()
        plan = F.FpsaPlan(grid, tile, win, H, d)
        plan.quantize(xx, xx, xx, "lhd", tile_order=not nat)
        torch.cuda.synchronize()
        xt = x.float().cpu().numpy()[perm, 0, :]
        c, s = O.quantize_qk_tilewise(xt, tv)
        got = plan.q_scales.cpu().numpy()
        print(dt, "natural" if nat else "tile", "scales ok", np.array_equal(got, s), got[:4], s[:4])
