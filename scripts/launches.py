"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg.setdefault(r[ki].split("(")[0][-40:], []).append(float(r[vi].replace(",", "")) / 1e3)
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print(f"{k:42s} n={len(v):5d} mean_us={sum(v)/len(v):10.2f} total_us={sum(v):11.1f} share={sum(v)/tot:6.1%}")
