"""Pipe utilisation per profiled launch of an .ncu-rep (--set full) -> JSON.

usage: python tools/pipe_util.py rep.ncu-rep out.json "<command that produced it>"
Keys: FP64 /
FMA (IMAD) / ALU / LSU instruction-issue shares of their pipes' peaks, issue
active, and the duration: the NTT passes' real bound is the FP64 pipe plus
latency, not HBM.
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(raw))
hdr, units = rows[0], dict(zip(rows[0], rows[1]))
KEYS = {
    "fp64_inst_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "fma_imad_inst_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "alu_inst_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "lsu_inst_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
}
per = defaultdict(list)
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    e = {}
    for k, m in KEYS.items():
        try:
            e[k] = float(d.get(m, "nan"))
        except ValueError:
            e[k] = None
    try:
        dur = float(d["gpu__time_duration.sum"]) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(
            units.get("gpu__time_duration.sum"), 1.0)
    except (KeyError, ValueError):
        dur = None
    e["duration_us"] = dur
    per[name].append(e)
out = []
for name, es in per.items():
    avg = {k: round(sum(x[k] for x in es if x[k] is not None) / max(1, sum(x[k] is not None for x in es)), 2)
           for k in es[0]}
    out.append({"kernel": name, "launches": len(es), **avg})
json.dump({"command": sys.argv[3] if len(sys.argv) > 3 else "", "kernels": out}, open(sys.argv[2], "w"), indent=1)
for e in out:
    print(e)
