#!/usr/bin/env python
"""Summarise one kernel of an ncu report: duration, DRAM bytes/throughput, occupancy,
top warp-stall reasons and the hottest SASS windows.  Usage: ncu_summary.py REPORT [REGEX]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__cluster_dim_x"]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if pat and not pat.search(name):
        continue
    print("==", name[:120])
    for w in want:
        if w in hdr:
            print(f"  {w:55s} {r[hdr.index(w)]} {rows[1][hdr.index(w)]}")
    st = [(float(r[i] or 0), h) for i, h in enumerate(hdr)
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    tot = sum(v for v, _ in st) or 1
    for v, h in sorted(st, reverse=True)[:8]:
        print(f"  stall {h[33:]:30s} {100 * v / tot:5.1f}%")
