"""Check the tv % 16 == 8 tail handling: per-row scale of the kernel output against the emulation."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
from conftest import golden_cases
import paper_2506_04648_b200 as fpsa
att = np.load("tests/golden/attention_cases.npz")
for name in ["tv120_d128", "tv240_d128", "c0_toy"]:
    c = golden_cases(att)[name]
    L = c["grid"][0] * c["grid"][1] * c["grid"][2]
    tv = c["tile"][0] * c["tile"][1] * c["tile"][2]
    q, k, v = O.gen_inputs(c["seed"], 1, 0, L, c["d"], c["dist"])
    tmap = fpsa.build_tile_map(fpsa.GridShape(*c["grid"], c["d"]), fpsa.TileScheme(*c["tile"]))
    out = fpsa.fp8_sparse_forward(fpsa.AttentionInputs(q, k, v, tmap), fpsa.ForwardConfig(window=fpsa.WindowSpec(*c["window"])))
    offs, ids = O.window_lists(O.tile_grid_dims(c["grid"], c["tile"]), c["window"])
    _, codes = O.fp8_sparse_forward(q, k, v, tv, offs, ids, O.FORMATS[c["fmt"]])
    emu = O.onepass_forward(codes, tv, offs, ids, O.FORMATS[c["fmt"]], tau=8.0, poly=True)
    ratio = (out * emu).sum(1) / (emu * emu).sum(1)
    print(name, "tv", tv, "cos", O.cosine(out, emu), "max-abs", O.max_abs(out, emu), "row scale min/max", ratio.min(), ratio.max())
