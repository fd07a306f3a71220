"""Per-region stall breakdown of an ncu source page (SASS).

  ncu -i rep --page source --csv --print-source sass > /tmp/s.csv
  python tools/sass_stalls.py /tmp/s.csv [--top 40]
Prints total stall reasons, and the hottest instructions with their dominant stalls.
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
h = rows[1]
data = rows[2:]
isrc, iss, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
ri = [h.index(x) for x in reasons]
tot = collections.Counter()
for r in data:
    for name, i in zip(reasons, ri):
        tot[name] += int(r[i] or 0)
S = sum(tot.values())
print("stall totals:", ", ".join(f"{k[6:]}={v / S * 100:.1f}%" for k, v in tot.most_common(12)))
top = sorted(data, key=lambda r: -int(r[iss] or 0))[:top_n]
for r in top:
    st = sorted(((int(r[i] or 0), n[6:]) for n, i in zip(reasons, ri)), reverse=True)[:3]
    print(f"{int(r[iss]) / S * 100:5.2f}% ex={int(r[iex]) / 1e6:7.1f}M {r[isrc].strip()[:60]:60s} " +
          " ".join(f"{n}={v}" for v, n in st))
