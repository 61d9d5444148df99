#!/usr/bin/env python
"""Per-instruction stall columns of one ncu report: top sites for a given stall reason.

  python tools/ncu_noinst.py gpurun_out/prof.ncu-rep [stall_no_inst] [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    col = sys.argv[2] if len(sys.argv) > 2 else "stall_no_inst"
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    ic, isrc = hdr.index(col), hdr.index("Source")
    data = [(int(r[ic] or 0), i, r[isrc].strip()) for i, r in enumerate(rows[2:]) if len(r) == len(hdr) and r[ic].isdigit()]
    tot = sum(d[0] for d in data)
    print(f"{col}: total {tot}")
    for v, i, s in sorted(data, reverse=True)[:n]:
        print(f"{v:7d} #{i:5d} {s[:80]}")


if __name__ == "__main__":
    main()
