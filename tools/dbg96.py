import sys, os, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import oracle as O
import paper_2506_04648_b200 as fpsa
d = int(sys.argv[1]); mode = sys.argv[2]
grid, tile, win = (6, 8, 8), (3, 4, 4), (3, 3, 3)
L = 6 * 8 * 8
q, k, v = O.gen_inputs(2, 1, 0, L, d)
tmap = fpsa.build_tile_map(fpsa.GridShape(*grid, d), fpsa.TileScheme(*tile))
t = time.time()
cfg = fpsa.ForwardConfig(window=fpsa.WindowSpec(*win), passthrough=(mode == "pt"), p_mode=("onepass" if mode == "one" else "normalized"))
out = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap), cfg)
torch.cuda.synchronize()
print(d, mode, "ok", time.time() - t, flush=True)
