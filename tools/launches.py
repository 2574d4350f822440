"""Summarize an ncu --csv launch list: mean per kernel and metric."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
ui = h.index("Metric Unit")
agg = defaultdict(list)
unit = {}
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg[(r[ki][:70], r[mi])].append(float(r[vi].replace(",", "")))
        unit[(r[ki][:70], r[mi])] = r[ui]
for k, v in sorted(agg.items()):
    print(f"{len(v):4d}  {sum(v) / len(v):14.1f} {unit[k]:8s} {k[1]:55s} {k[0]}")
