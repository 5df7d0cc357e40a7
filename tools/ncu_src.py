"""Per-instruction stall samples of one kernel from `ncu --page source --csv --print-source sass`.
usage: python tools/ncu_src.py src.csv <kernel index (0-based)> [top]"""
import csv
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
starts = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
k = int(sys.argv[2])
top_n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
block = lines[starts[k]:starts[k + 1]]
print(block[0][:150])
rows = list(csv.reader(block[1:]))
hdr = rows[0]
data = [dict(zip(hdr, r)) for r in rows[1:] if len(r) == len(hdr)]
S = "Warp Stall Sampling (All Samples)"
tot = sum(int(d[S] or 0) for d in data)
print("instructions", len(data), "samples", tot)
ops = Counter()
for d in data:
    toks = d["Source"].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    ops[op.split(".")[0]] += int(d[S] or 0)
print("by opcode:", ", ".join(f"{o}={100 * v / tot:.1f}%" for o, v in ops.most_common(12)))
for idx, d in sorted(enumerate(data), key=lambda x: -int(x[1][S] or 0))[:top_n]:
    print(f"{idx:5d} {100 * int(d[S] or 0) / tot:5.1f}%  {d['Source'][:80]}")
