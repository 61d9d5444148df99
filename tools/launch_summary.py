#!/usr/bin/env python
"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): per kernel the launch count,
mean and total device time and share; plus the launches of the LAST timed bench step in order.

  python tools/launch_summary.py gpurun_out/r01_launches.csv [launches_per_step]
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    iN, iM, iV, iId = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    launches = []
    for r in rows[start + 1:]:
        if len(r) > iV and r[iM] == "gpu__time_duration.sum":
            v = float(r[iV].replace(",", ""))
            name = r[iN].split("(")[0].replace("void ", "").replace("wl::<unnamed>::", "")
            launches.append((int(r[iId]), name, v / 1e3))  # ns -> us
    agg = collections.defaultdict(list)
    for _, n, us in launches:
        agg[n].append(us)
    tot = sum(sum(v) for v in agg.values())
    print("# per-kernel launch count, mean and total device time (us; cold-cache, serialised: compare shares)")
    for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):5d} {sum(v) / len(v):10.1f} {sum(v):12.1f} {100 * sum(v) / tot:5.1f}%  {n}")
    if len(sys.argv) > 2:
        k = int(sys.argv[2])
        step = launches[-k:]
        st = sum(us for _, _, us in step)
        print(f"\n# the last {k} launches (one step), in order; sum {st:.1f} us")
        for i, n, us in step:
            print(f"{i:5d} {us:9.1f} {100 * us / st:5.1f}%  {n}")


if __name__ == "__main__":
    main()
