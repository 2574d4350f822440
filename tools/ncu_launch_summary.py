"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: total
time per kernel (name + template args), launch count, share."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = collections.defaultdict(float)
cnt = collections.Counter()
n = 0
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    n += 1
    if n <= skip:
        continue
    name = r[ki]
    name = name.replace("dsx_nn::", "").replace("(anonymous namespace)::", "")
    name = name.split("(CUtensorMap")[0].split("(const")[0].split("(float")[0]
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
s = sum(tot.values())
print(f"{n - skip} launches, {s / 1e6:.3f} ms total (ncu serialised, cold-cache)")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / 1e6:9.3f} ms {100 * v / s:5.1f}%  x{cnt[k]:4d}  {k[:150]}")
