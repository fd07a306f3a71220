"""Quantiser timing at a BASELINE config: FpsaPlan.quantize (q, k, v of bf16 [L, H, d], natural order) and
the amax-hook variant, CUDA events over N calls.  Prints ms and algorithmic GB/s (9 B per element)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_04648_b200 as fpsa  # noqa: E402

grid, tile, H, d = (21, 45, 80), (3, 5, 16), int(os.environ.get("H", "40")), 128
L = grid[0] * grid[1] * grid[2]
gen = torch.Generator(device="cuda").manual_seed(0)
xs = [torch.randn((L, H, d), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(3)]
plan = fpsa.FpsaPlan(grid, tile, (5, 5, 3), H, d)
va = xs[2].float().abs().amax(dim=0).contiguous()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, n=20):
    for _ in range(3):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for s, e in ev:
        flush.zero_()
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return sorted(s.elapsed_time(e) for s, e in ev)[n // 2]


algo = 9 * L * H * d
res = {}
for name, fn in (("quantize", lambda: plan.quantize(*xs, "lhd")),
                 ("quantize_with_v_amax", lambda: plan.quantize_with_amax(*xs, None, None, va, layout="lhd"))):
    ms = timed(fn)
    res[name] = {"ms": ms, "GBps": algo / ms / 1e6}
print(json.dumps({"config": "wan14b_720p", "heads": H, "algorithmic_bytes": algo, **res}))
