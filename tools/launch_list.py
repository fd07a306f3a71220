"""Compact an ncu launch list (--metrics gpu__time_duration.sum --csv) into profiles/.

  python tools/launch_list.py gpurun_out/launches.csv profiles/rNN_launches.csv
Also prints each kernel family's share of the summed device time.
"""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
ik, iv, ig, ib = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size"), h.index("Block Size")
share = collections.Counter()
with open(sys.argv[2], "w") as f:
    f.write("id,kernel,grid,block,gpu__time_duration_ns\n")
    for r in rows[1:]:
        name = r[ik]
        short = name.replace("void ", "").split("(")[0]
        short = short.split("<")[0] if "fpsa" not in short else short
        short = short.replace("fpsa::<unnamed>::", "")[:70]
        ns = float(r[iv].replace(",", ""))
        share[short] += ns
        f.write(f'{r[0]},"{short}","{r[ig]}","{r[ib]}",{ns:.0f}\n')
tot = sum(share.values())
for k, v in share.most_common():
    print(f"{v / tot * 100:5.1f}%  {v / 1e6:8.3f} ms  {k}")
