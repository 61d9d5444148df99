#!/usr/bin/env python
"""Instruction mix per barrier-delimited SASS segment + top stall reasons of one kernel.

  python tools/ncu_segments.py gpurun_out/prof.ncu-rep [kernel-regex]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kflag = ["-k", f"regex:{sys.argv[2]}"] if len(sys.argv) > 2 else []
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", *kflag],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    ins = [(r[iS].strip(), int(r[iE] or 0), int(r[iW] or 0)) for r in rows[2:] if len(r) == len(hdr) and r[iE].isdigit()]
    segs, cur = [], []
    for s, e, w in ins:
        cur.append((s, e, w))
        if "BAR.SYNC" in s:
            segs.append(cur)
            cur = []
    segs.append(cur)
    for i, sg in enumerate(segs):
        tot = sum(x[1] for x in sg)
        if tot < 1e5:
            continue
        ff = sum(x[1] for x in sg if "FFMA2" in x[0])
        st = sum(x[2] for x in sg)
        ops = collections.Counter()
        for s, e, w in sg:
            op = s.split()[0]
            if op.startswith("@"):
                op = s.split()[1]
            ops[op.split(".")[0]] += e
        print(f"seg {i}: instr {tot / 1e6:7.2f}M FFMA2 {ff / 1e6:6.2f}M stall {st:6d} | " +
              ", ".join(f"{k}:{v / 1e6:.2f}" for k, v in ops.most_common(9)))
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", *kflag], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, v = r[0], r[2]
    items = [(h[i].split("stalled_")[1], v[i]) for i in range(len(h))
             if "smsp__pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued")]
    items.sort(key=lambda x: -float(x[1] or 0))
    print("stalls: " + " ".join(f"{k}={x}" for k, x in items[:9]))


if __name__ == "__main__":
    main()
