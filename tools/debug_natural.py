import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O
import paper_2506_04648_b200 as F
grid, tile, win, H, d = (6, 10, 32), (3, 5, 16), (3, 3, 3), 3, 128
L = 1920; tv = 240
g = torch.Generator(device="cuda").manual_seed(1)
q, k, v = (torch.randn((L, H, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
plan = F.FpsaPlan(grid, tile, win, H, d)
plan.quantize(q, k, v, "lhd")
torch.cuda.synchronize()
perm = O.tile_perm(grid, tile)
M = plan.M
for name, x, codes, scales in (("q", q, plan.q_codes, plan.q_scales), ("k", k, plan.k_codes, plan.k_scales), ("v", v, plan.v_codes, plan.v_scales)):
    cc = codes.view(H, M, plan.pitch, d).cpu().numpy()
    xs = x.float().cpu().numpy()
    for h in range(H):
        xt = xs[perm, h, :]
        if name == "v":
            c, s = O.quantize_v_channelwise(xt); sc = scales.view(H, d)[h].cpu().numpy()
        else:
            c, s = O.quantize_qk_tilewise(xt, tv); sc = scales.view(H, M)[h].cpu().numpy()
        print(name, h, "scales", np.array_equal(sc, s), "codes", np.array_equal(cc[h, :, :tv].reshape(L, d), c))
out = torch.empty((L, H, d), dtype=torch.float32, device="cuda")
plan.attention(out, "lhd")
out_t = torch.empty((L, H, d), dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
for h in range(H):
    p1 = F.FpsaPlan(grid, tile, win, 1, d)
    qt, kt, vt = (x[:, h, :].float()[perm].contiguous() for x in (q, k, v))
    p1.quantize(qt, kt, vt, "ld", tile_order=True)
    o1 = torch.empty((L, d), dtype=torch.float32, device="cuda")
    p1.attention(o1, "ld", tile_order=True)
    torch.cuda.synchronize()
    same_codes = [torch.equal(a.view(M, -1, d)[:, :tv], b.view(H, M, -1, d)[h, :, :tv]) for a, b in ((p1.q_codes, plan.q_codes), (p1.k_codes, plan.k_codes), (p1.v_codes, plan.v_codes))]
    d_out = (out[:, h, :][perm] - o1).abs().max().item()
    print("head", h, "codes equal", same_codes, "max diff", d_out)
    # natural order attention from the 1-head plan
    o2 = torch.empty((L, d), dtype=torch.float32, device="cuda")
    p1.attention(o2, "ld", tile_order=False)
    torch.cuda.synchronize()
    print("   natural vs tile (same codes):", (o2[perm] - o1).abs().max().item())
