"""Per-kernel share of an ncu --csv launch list (gpu__time_duration.sum only).

usage: python tools/launch_share.py launches.csv [top]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")
    v = float(d["Metric Value"].replace(",", ""))
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(t for _, t in agg.values())
print(f"total {tot / 1e3:.3f} ms over {sum(n for n, _ in agg.values())} launches (serialised, cold caches)")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{n:6d} {t:10.1f} us {100 * t / tot:5.1f}%  {k[:70]}")
