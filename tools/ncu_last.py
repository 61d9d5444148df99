#!/usr/bin/env python
"""Print the last N launches (kernel, us, DRAM MB) of an ncu --csv metrics log:  python tools/ncu_last.py log.csv N"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
iN, iM, iV, iId = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
by = {}
for r in rows[start + 1:]:
    if len(r) > iV:
        d = by.setdefault(int(r[iId]), {"name": r[iN].split("(")[0].replace("void ", "").replace("wl::<unnamed>::", "")})
        d[r[iM]] = float(r[iV].replace(",", ""))
ids = sorted(by)[-int(sys.argv[2]):]
tot = 0.0
for i in ids:
    d = by[i]
    us = d.get("gpu__time_duration.sum", 0) / 1e3
    tot += us
    mb = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
    print(f"{d['name'][:60]:60s} {us:8.1f} us {mb:8.1f} MB")
print(f"total {tot:.1f} us")
