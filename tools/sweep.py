"""BASELINE config 5: the 50-step schedule at the Wan2.1-14B 720p shape.

  python tools/sweep.py [--steps 50] [--no-graphs] [--fidelity] [--csv gpurun_out/sweep_c4.csv]
Prints one JSON line (total ms, per-regime mean ms and effective TFLOPS) and
writes the per-step CSV (reference schema + ms, eff_tflops).  --fidelity also
fills cosine / mse / snr per step against the full-precision passthrough
kernel (untimed).
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2506_04648_b200.schedule_runner import ScheduleRunner, c4_schedule, rows_to_csv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--no-graphs", action="store_true")
ap.add_argument("--fidelity", action="store_true")
ap.add_argument("--csv", default="gpurun_out/sweep_c4.csv")
args = ap.parse_args()
grid, H, d = (21, 45, 80), 40, 128
L = grid[0] * grid[1] * grid[2]
gen = torch.Generator(device="cuda").manual_seed(5)
q, k, v = (torch.randn((L, H, d), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
runner = ScheduleRunner(grid, c4_schedule(args.steps), H, d, use_graphs=not args.no_graphs, fidelity=args.fidelity)
for t in (1, args.steps // 2, args.steps):  # build plans / graphs of every regime
    runner.step(t, q, k, v, out)
torch.cuda.synchronize()
rows = runner.run(q, k, v, out)
os.makedirs(os.path.dirname(args.csv) or ".", exist_ok=True)
with open(args.csv, "w") as f:
    f.write(rows_to_csv(rows))
summary = {"metric": "C4 schedule sweep, Wan2.1-14B 720p, 40 heads, per-step quantise + attention",
           "steps": len(rows), "total_ms": sum(r.ms for r in rows), "graphs": not args.no_graphs,
           "fidelity": args.fidelity}
for regime in ("early", "mid", "late"):
    rr = [r for r in rows if r.regime == regime]
    if rr:
        summary[regime] = {"steps": len(rr), "tile": rr[0].tile, "window": rr[0].window,
                           "density": rr[0].density, "mean_ms": statistics.mean(r.ms for r in rr),
                           "eff_tflops": statistics.mean(r.eff_tflops for r in rr)}
        if args.fidelity:
            summary[regime].update(cosine_sim=min(r.cosine_sim for r in rr), snr_db=min(r.snr_db for r in rr))
print(json.dumps(summary))
