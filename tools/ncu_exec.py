"""Executed-instruction counts by opcode of one kernel from `ncu --page source --csv --print-source sass`.
usage: python tools/ncu_exec.py src.csv <kernel index (0-based)>"""
import csv
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
starts = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
k = int(sys.argv[2])
block = lines[starts[k]:starts[k + 1]]
print(block[0][:150])
rows = list(csv.reader(block[1:]))
hdr = rows[0]
data = [dict(zip(hdr, r)) for r in rows[1:] if len(r) == len(hdr)]
col = next(c for c in hdr if c.startswith("# Instructions Executed") or c == "Instructions Executed")
ops, tot = Counter(), 0
for d in data:
    toks = d["Source"].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    n = int(d[col] or 0)
    ops[op.split(".")[0] + ("." + op.split(".")[1] if op.startswith("IMAD") and "." in op else "")] += n
    tot += n
print("warp instructions executed", tot, "static", len(data), "columns", [c for c in hdr if "Instr" in c][:4])
print(", ".join(f"{o}={100 * v / tot:.1f}%" for o, v in ops.most_common(16)))
