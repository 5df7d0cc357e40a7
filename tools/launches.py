"""Summarise an ncu --csv launch list: per-kernel time share of the second half."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
part = data[int(len(data) * (1 - frac)):]
agg = defaultdict(lambda: [0, 0.0])
for d in part:
    agg[d["Kernel Name"][:72]][0] += 1
    agg[d["Kernel Name"][:72]][1] += float(d["Metric Value"])
tot = sum(v for c, v in agg.values())
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
    print(f"{c:6d} {v / 1e3:10.1f} us {100 * v / tot:5.1f}%  {k}")
print(f"total {tot / 1e6:.3f} ms over {len(part)} launches")
