"""One line per profiled launch from an .ncu-rep raw CSV export."""
import csv
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(raw))
hdr, units = rows[0], dict(zip(rows[0], rows[1]))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
for r in rows[2:]:
    d = dict(zip(hdr, r))

    def f(k):
        try:
            return float(d.get(k, "nan") or "nan") * SCALE.get(units.get(k, ""), 1.0)
        except ValueError:
            return float("nan")
    dur = f("gpu__time_duration.sum")
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    print(f"{d['Kernel Name'][:60]:60s} grid={d['Grid Size']:>14} dur={dur:8.1f}us "
          f"regs={d.get('launch__registers_per_thread')} occ={f('sm__warps_active.avg.pct_of_peak_sustained_active'):4.0f}% "
          f"issue={f('smsp__issue_active.avg.pct_of_peak_sustained_active'):4.0f}% "
          f"dram={(rd + wr) / 1e6:8.1f}MB ({(rd + wr) / dur / 1e3:6.0f} GB/s) "
          f"inst={f('smsp__inst_executed.sum') / 1e6:6.2f}M")
    stalls = []
    for k in hdr:
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                stalls.append((float(d[k]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1
    print("      stalls: " + ", ".join(f"{k}={100 * v / tot:.0f}%" for v, k in sorted(stalls, reverse=True)[:6]))
