#!/usr/bin/env python
"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*
--csv): launches, total time, share of the list, DRAM bytes per launch.
Usage: launch_list.py LAUNCHES.csv [first_id]"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr, rows = rows[0], rows[1:]
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
k = {h: i for i, h in enumerate(hdr)}
per = collections.defaultdict(lambda: collections.defaultdict(float))
for r in rows:
    if int(r[k["ID"]]) < first:
        continue
    name = re.sub(r"\(.*$", "", r[k["Kernel Name"]]).replace("(anonymous namespace)::", "").replace("fg::", "")
    name = re.sub(r"^.*::", "", name) if "lam_gemm" not in name else name.split("::")[-1]
    per[(name, r[k["ID"]])][r[k["Metric Name"]]] = float(r[k["Metric Value"]].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (name, _), m in per.items():
    a = agg[name]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
for name, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{name[:44]:44s} launches {n:4d} total {t:14.1f} share {100 * t / tot:5.1f}%  dram/launch {b / n / 1e9:7.3f} GB")
