"""Top source lines by warp-state samples from `ncu -i rep --page source --csv --print-source cuda`."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
for i, r in enumerate(rows):
    if "Source" in r and any("Sampl" in c for c in r):
        hdr = i
        break
if hdr is None:
    print(out[:3000])
    sys.exit(0)
h = rows[hdr]
si = h.index("Source")
cols = [i for i, c in enumerate(h) if "Sampl" in c]
print("columns:", [h[i] for i in cols])
data = []
for r in rows[hdr + 1:]:
    if len(r) <= max(cols):
        continue
    try:
        v = float(r[cols[0]] or 0)
    except ValueError:
        continue
    data.append((v, r[0] if r else "", r[si][:140], [r[i] for i in cols]))
tot = sum(d[0] for d in data) or 1
for v, ln, src, allv in sorted(data, key=lambda x: -x[0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100 * v / tot:5.1f}%  L{ln:>5}  {src}  {allv}")
