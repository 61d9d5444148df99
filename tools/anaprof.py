#!/usr/bin/env python
"""Per-run timing of one analysis level (debug build with -DWL_ANA_PROFILE, loaded via WL_LIB): run durations by
band height and strip, per-SM finish times.  python tools/anaprof.py --cfg 5 --level 2"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1707_02018_b200 import inputs, wl
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=5)
    ap.add_argument("--level", type=int, default=1)
    ap.add_argument("--size", type=int, default=0, help="square input of this size instead of the config's level")
    ap.add_argument("--brief", action="store_true")
    ap.add_argument("--chain", type=int, default=0, help="run a J-level W* chain on the config's image; the profile is level J's")
    a = ap.parse_args()
    c = inputs.CONFIGS[a.cfg]
    # the level's input size: run a 1-level plan on an image of that size
    full = wl.Plan(c.h, c.w, c.levels, c.filt, c.bc, c.dtype)
    h, w = full.chain_h[a.level - 1], full.chain_w[a.level - 1]
    if a.size:
        h = w = a.size
    plan = wl.Plan(h, w, 1, c.filt, c.bc, c.dtype)
    if a.chain:
        h, w = c.h, c.w
        plan = wl.Plan(h, w, a.chain, c.filt, c.bc, c.dtype)
    img = torch.randn(c.batch, h, w, device="cuda", dtype=plan.torch_dtype)
    out = torch.empty(c.batch, plan.p_alloc, device="cuda", dtype=plan.torch_dtype)
    ws = plan._ws(wl.OP_ADJOINT, c.batch)
    for _ in range(3):
        plan.adjoint(img, out=out, ws=ws)
    torch.cuda.synchronize()
    L = wl.lib()
    buf = np.zeros((8192, 4), dtype=np.uint64)
    L.wl_debug_ana_prof(buf.ctypes.data_as(ctypes.c_void_p), 8192)
    used = buf[:, 1] > 0
    t0, t1, sm, meta = buf[used, 0].astype(np.int64), buf[used, 1].astype(np.int64), buf[used, 2], buf[used, 3]
    base = t0.min()
    start, end = (t0 - base) / 1e3, (t1 - base) / 1e3
    dur = end - start
    col = (meta >> np.uint64(32)).astype(int)
    rows = (meta & np.uint64(0xffffffff)).astype(int)
    print(f"input {h}x{w}: runs {used.sum()}  span {end.max():.1f} us  starts {start.min():.1f}..{start.max():.1f}  "
          f"run duration min/median/max {dur.min():.1f} / {np.median(dur):.1f} / {dur.max():.1f} us")
    ncols = col.max() + 1
    if a.brief:
        nstrips = ncols // c.batch
        strip = col % nstrips
        big = rows == rows.max()
        print(f"  size {h}: span {end.max():.1f}; rows {rows.max()} runs: interior median {np.median(dur[big & (strip < nstrips - 1)]):.1f}, "
              f"last strip median {np.median(dur[big & (strip == nstrips - 1)]):.1f}")
        return
    nstrips = ncols // c.batch
    strip = col % nstrips
    for r in sorted(set(rows)):
        m = rows == r
        print(f"band {r} rows: {m.sum()} runs, dur median {np.median(dur[m]):.1f} max {dur[m].max():.1f}, end median {np.median(end[m]):.1f} max {end[m].max():.1f}")
    for sname, m in (("first", strip == 0), ("last", strip == nstrips - 1), ("interior", (strip > 0) & (strip < nstrips - 1))):
        if m.any():
            print(f"{sname} strip: {m.sum()} runs, dur median {np.median(dur[m]):.1f} max {dur[m].max():.1f}")
    for r in sorted(set(rows)):
        line = " ".join(f"{np.median(dur[(rows == r) & (strip == st)]):.1f}" if ((rows == r) & (strip == st)).any() else "-"
                        for st in range(nstrips))
        print(f"per-strip median dur, band {r}: {line}")
    smend, smcnt = {}, {}
    for k in range(len(sm)):
        smend[int(sm[k])] = max(smend.get(int(sm[k]), 0), end[k])
        smcnt[int(sm[k])] = smcnt.get(int(sm[k]), 0) + 1
    v = np.array(sorted(smend.values()))
    print(f"SMs {len(v)}  finish: min {v.min():.1f} p25 {np.percentile(v,25):.1f} median {np.median(v):.1f} p75 {np.percentile(v,75):.1f} max {v.max():.1f} us; CTAs/SM {min(smcnt.values())}..{max(smcnt.values())}")
    slow = sorted(range(len(dur)), key=lambda k: -end[k])[:10]
    for k in slow:
        print(f"  last: end {end[k]:.1f} dur {dur[k]:.1f} start {start[k]:.1f} sm {int(sm[k])} img {col[k] // nstrips} strip {strip[k]} rows {rows[k]}")


if __name__ == "__main__":
    main()
