#!/usr/bin/env python
"""Per-CUDA-source-line instruction counts and stall samples of one kernel in an ncu report
(needs -lineinfo builds and --import-source).  Inlined code is attributed to the line of the
callee (e.g. the fma2 helper), so lines are also grouped by the SASS opcode class.

  python tools/ncu_lines.py gpurun_out/prof.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = None
    res = []
    cur = None
    for r in rows:
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            iE = hdr.index("Instructions Executed")
            iW = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0]:
            cur = [int(r[0]), r[1].strip()[:100], int(r[iE] or 0) if r[iE].isdigit() else 0,
                   int(r[iW] or 0) if r[iW].isdigit() else 0]
            res.append(cur)
    tot = sum(x[2] for x in res) or 1
    print(f"total {tot}")
    for ln, src, e, w in sorted(res, key=lambda x: -x[2])[:top]:
        print(f"{e:11d} {100 * e / tot:5.1f}% stall {w:6d}  L{ln:<4d} {src}")


if __name__ == "__main__":
    main()
