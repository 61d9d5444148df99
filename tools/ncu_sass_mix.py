#!/usr/bin/env python
"""Dynamic SASS instruction mix and top stall sites of one kernel in an ncu report.

  python tools/ncu_sass_mix.py gpurun_out/prof.ncu-rep [kernel-substring]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if len(sys.argv) > 2:
        cmd += ["-k", f"regex:{sys.argv[2]}"]
    txt = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    mix = collections.Counter()
    stall = collections.Counter()
    sites = []
    tot = 0
    for r in rows[2:]:
        if len(r) < len(hdr) or not r[iE].isdigit():
            continue
        src = r[iS].strip()
        op = src.split()[0]
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        e, w = int(r[iE]), int(r[iW] or 0)
        mix[op] += e
        stall[op] += w
        tot += e
        sites.append((w, r[0], src[:90]))
    print(f"total warp instructions {tot}")
    for op, e in mix.most_common(30):
        print(f"  {op:10s} {e:12d} {100 * e / tot:5.1f}%  stall-samples {stall[op]}")
    print("top stall sites:")
    for w, a, s in sorted(sites, reverse=True)[:15]:
        print(f"  {w:6d} {a} {s}")


if __name__ == "__main__":
    try:
        main()
    except BrokenPipeError:  # output cut short by `head`
        pass
