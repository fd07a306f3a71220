"""Full-precision passthrough path (bf16 tcgen05 kind::f16) at a BASELINE video shape, one GPU.

  python tools/bench_passthrough.py [--config wan14b_720p] [--steps 10] [--warmup 3]
One JSON line: gather (natural bf16 -> tile-major bf16) and attention ms,
effective TFLOP/s of the attention kernel against the measured bf16 dense
peak (MEASURED_PEAKS.json), and its fidelity against nothing (it IS the
reference); plus the FP8 path's fidelity against it on the same inputs.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_04648_b200 as fpsa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="wan14b_720p", choices=sorted(bench.CONFIGS))
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
args = ap.parse_args()
grid, H, d, tile, win = bench.CONFIGS[args.config]
L = grid[0] * grid[1] * grid[2]
gen = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((L, H, d), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty((L, H, d), dtype=torch.bfloat16, device="cuda")
plan = fpsa.PassthroughPlan(grid, tile, win, H, d)
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")  # > L2
tg, ta = [], []
for i in range(args.warmup + args.steps):
    flush.zero_()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    plan.gather(q, k, v, "lhd")
    e[1].record()
    plan.attention(out, "lhd")
    e[2].record()
    torch.cuda.synchronize()
    if i >= args.warmup:
        tg.append(e[0].elapsed_time(e[1]))
        ta.append(e[1].elapsed_time(e[2]))
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
ms_a = statistics.median(ta)
tf = plan.flops / (ms_a * 1e-3) / 1e12
ref = torch.empty((L, H, d), dtype=torch.float32, device="cuda")
plan(q, k, v, "lhd", out=ref)
fp8 = fpsa.FpsaPlan(grid, tile, win, H, d)(q, k, v, "lhd", out_dtype=torch.float32)
fid = fpsa.device_fidelity(ref, fp8, "lhd")
print(json.dumps({
    "metric": "passthrough (bf16 operands, f32 softmax) sparse attention", "config": args.config,
    "grid": grid, "heads": H, "tile": tile, "window": win, "steps": args.steps,
    "gather_ms": statistics.median(tg), "attn_ms": ms_a, "attn_tflops": tf,
    "bf16_peak_tflops": peaks["bf16_tflops"], "frac_bf16_peak": tf / peaks["bf16_tflops"],
    "bf16_spec_tflops": 2250.0, "redo_items": plan.redo_count(),
    "fp8_vs_passthrough": {"cosine_min": min(m[0] for m in fid), "snr_db_min": min(m[2] for m in fid),
                           "mse_mean": sum(m[1] for m in fid) / len(fid)},
}))
