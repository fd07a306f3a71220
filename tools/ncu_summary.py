"""Summarise an ncu report (--set full) into the numbers the roofline needs.

  python tools/ncu_summary.py gpurun_out/attn.ncu-rep [--json out.json] [--algo-bytes B]

Prints per launch: kernel, duration, SM clock, DRAM bytes read/write, tensor
pipe / XU (MUFU) / FMA utilisation, registers, local-memory traffic,
achieved occupancy and the top stall reasons.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    ("duration", r"^gpu__time_duration\.sum$"),
    ("sm_clock", r"^smsp__cycles_elapsed\.avg\.per_second$"),
    ("dram_read", r"^dram__bytes_read\.sum$"),
    ("dram_write", r"^dram__bytes_write\.sum$"),
    ("dram_pct", r"^gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed$"),
    ("tensor_pipe_pct", r"^sm__pipe_tensor_cycles_active\.avg\.pct_of_peak_sustained_elapsed$"),
    ("tensor_pipe_rt_pct", r"^TPC\.TriageCompute\.sm__pipe_tensor_cycles_active_realtime\.avg\.pct_of_peak_sustained_elapsed$"),
    ("xu_pipe_pct", r"^sm__inst_executed_pipe_xu\.avg\.pct_of_peak_sustained_active$"),
    ("fma_pipe_pct", r"^sm__inst_executed_pipe_fma\.avg\.pct_of_peak_sustained_active$"),
    ("alu_pipe_pct", r"^sm__inst_executed_pipe_alu\.avg\.pct_of_peak_sustained_active$"),
    ("issue_active_pct", r"^sm__inst_issued\.avg\.pct_of_peak_sustained_active$"),
    ("registers", r"^launch__registers_per_thread$"),
    ("local_ld_sectors", r"^l1tex__t_sectors_pipe_lsu_mem_local_op_ld\.sum$"),
    ("local_st_sectors", r"^l1tex__t_sectors_pipe_lsu_mem_local_op_st\.sum$"),
    ("occupancy_pct", r"^sm__warps_active\.avg\.pct_of_peak_sustained_active$"),
    ("l2_hit_pct", r"^lts__t_sector_hit_rate\.pct$"),
    ("grid", r"^launch__grid_size$"),
    ("block", r"^launch__block_size$"),
    ("smem_dyn", r"^launch__shared_mem_per_block_dynamic$"),
]


def raw(report: str):
    txt = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    header, units, data = rows[0], rows[1], rows[2:]
    return header, units, data


def stalls(header, row):
    out = []
    for k, v in zip(header, row):
        m = re.match(r"^smsp__average_warp_latency_issue_stalled_(\w+)\.ratio$", k) or \
            re.match(r"^smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", k)
        if m:
            try:
                out.append((float(v), m.group(1)))
            except ValueError:
                pass
    return sorted(out, reverse=True)[:6]


def to_bytes(v: float, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return v * scale.get(unit, 1)


def to_seconds(v: float, unit: str) -> float:
    return v * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9,
                "second": 1.0}.get(unit, 1e-9)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--json")
    ap.add_argument("--algo-bytes", type=float, default=None)
    args = ap.parse_args()
    header, units, data = raw(args.report)
    idx = {k: i for i, k in enumerate(header)}
    name_i = idx.get("Kernel Name")
    results = []
    for row in data:
        rec = {"kernel": row[name_i][:120] if name_i is not None else "?"}
        for key, pat in KEYS:
            for k, i in idx.items():
                if re.match(pat, k):
                    val = row[i].replace(",", "")
                    try:
                        f = float(val)
                    except ValueError:
                        rec[key] = val
                        break
                    if key in ("dram_read", "dram_write"):
                        f = to_bytes(f, units[i])
                    elif key == "duration":
                        f = to_seconds(f, units[i])
                    rec[key] = f
                    break
        rec["dram_bytes"] = rec.get("dram_read", 0.0) + rec.get("dram_write", 0.0)
        rec["top_stalls"] = [f"{n}={v:.2f}" for v, n in stalls(header, row)]
        results.append(rec)
    for r in results:
        print(json.dumps(r))
    if args.json:
        with open(args.json, "w") as f:
            json.dump(results, f, indent=1)


if __name__ == "__main__":
    sys.exit(main())
