"""Aggregate an ncu --csv launch list (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum) into per-kernel achieved DRAM GB/s -> JSON.

usage: python tools/kernel_roofline.py launches.csv out.json "<command>"
"""
import csv
import json
import re
import sys
from collections import defaultdict

import os

_PEAKS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
PEAK = float(json.load(open(_PEAKS))["hbm_gbs"]) if os.path.exists(_PEAKS) else 6450.3  # measured copy GB/s
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = defaultdict(lambda: {"launches": 0, "s": 0.0, "bytes": 0.0})
cur = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (d["ID"], re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").strip())
    v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
    cur.setdefault(key, {})[d["Metric Name"]] = v
for (lid, name), m in cur.items():
    e = per[name]
    e["launches"] += 1
    e["s"] += m.get("gpu__time_duration.sum", 0.0)
    e["bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
total = sum(e["s"] for e in per.values())
out = []
for name, e in sorted(per.items(), key=lambda kv: -kv[1]["s"]):
    gbs = e["bytes"] / e["s"] / 1e9 if e["s"] else 0.0
    out.append({"kernel": name, "launches": e["launches"], "time_share": round(e["s"] / total, 4),
                "avg_us": round(e["s"] / e["launches"] * 1e6, 2), "dram_gb_per_s": round(gbs, 1),
                "frac_of_hbm": round(gbs / PEAK, 3)})
total_bytes = sum(e["bytes"] for e in per.values())
json.dump({"command": sys.argv[3] if len(sys.argv) > 3 else "", "peak_gbs": PEAK,
           "note": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                   "--clock-control none " + (sys.argv[4] if len(sys.argv) > 4 else "") + " (launches serialised)",
           "dram_bytes": int(total_bytes), "time_s": total,
           "kernels": out}, open(sys.argv[2], "w"), indent=1)
print(f"total: {total * 1e3:.3f} ms, DRAM {total_bytes / 1e9:.2f} GB")
for k in out:
    print(f"{k['kernel'][:60]:60s} {k['launches']:5d} {100 * k['time_share']:5.1f}% {k['avg_us']:8.1f}us "
          f"{k['dram_gb_per_s']:7.0f} GB/s {100 * k['frac_of_hbm']:5.1f}%")
