"""Share of the attention kernel's stall samples spent in the MMA warp's issue loop, from an ncu source page
(ncu -i REP --page source --csv --print-source sass). The loop is located from its UTCQMMA instructions: the
per-step MMAs are the ones executed most often; its instructions are those with the same execution count."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
ex = lambda r: int(r[col["Instructions Executed"]] or 0)
samp = lambda r: float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
mma = [i for i, r in enumerate(data) if "UTCQMMA" in r[col["Source"]]]
c = max(ex(data[i]) for i in mma)  # the steady-state step's MMAs
steady = [i for i in mma if ex(data[i]) >= 0.95 * c]
near = lambda i: 0.95 * c <= ex(data[i]) <= 1.05 * c or ex(data[i]) == 0
lo, hi = steady[0], steady[-1]
while lo > 0 and near(lo - 1):  # the loop body: contiguous code executed once per step
    lo -= 1
while hi + 1 < len(data) and near(hi + 1):
    hi += 1
loop = data[lo:hi + 1]
step_counts = {c}
total = sum(samp(r) for r in data)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.Counter()
for r in loop:
    for h in reasons:
        agg[h] += float(r[col[h]] or 0)
spin = max(loop, key=samp)
# the out-of-line retry stubs of the loop's barrier waits (try_wait spin) sit after the function body
print(f"kernel samples {total:.0f}; MMA-loop instructions {len(loop)} (executions per launch {sorted(step_counts)})")
print(f"MMA-loop samples {sum(samp(r) for r in loop):.0f} = {100 * sum(samp(r) for r in loop) / total:.1f} % of all "
      f"(12 warps per CTA: one warp always resident would be {100 / 12:.1f} %)")
print(f"largest single instruction (the p_ready wait loop): {samp(spin):.0f} samples: {spin[col['Source']][:60]}")
for h, v in agg.most_common(8):
    print(f"  {h:24s} {v:8.0f}")
