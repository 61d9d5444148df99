#!/usr/bin/env python
"""Per-run timing of the ring residual (debug build with -DWL_RING_PROFILE, loaded via WL_LIB):
per-SM busy time and the runs' spread.  python tools/ringprof.py"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1707_02018_b200 import inputs, wl
    c = inputs.CONFIGS[5]
    blur = wl.Blur(c.h, c.w, 15, 3.0, dtype="float32")
    u = torch.randn(4, c.h, c.w, device="cuda")
    b = torch.randn(4, c.h, c.w, device="cuda")
    s = torch.empty_like(u)
    for _ in range(3):
        blur.residual_adjoint(u, b, out=s)
    torch.cuda.synchronize()
    L = wl.lib()
    buf = np.zeros((8192, 4), dtype=np.uint64)
    L.wl_debug_ring_prof(buf.ctypes.data_as(ctypes.c_void_p), 8192)
    used = buf[:, 1] > 0
    t0, t1, sm, meta = buf[used, 0].astype(np.int64), buf[used, 1].astype(np.int64), buf[used, 2], buf[used, 3]
    base = t0.min()
    start, end = (t0 - base) / 1e3, (t1 - base) / 1e3
    dur = end - start
    col = (meta >> np.uint64(32)).astype(int)
    rows = (meta & np.uint64(0xffffffff)).astype(int)
    print(f"runs {used.sum()}  kernel span {end.max():.1f} us  run duration min/median/max {dur.min():.1f} / {np.median(dur):.1f} / {dur.max():.1f} us")
    nstrips = 17
    strip = col % nstrips
    edge = (strip == 0) | (strip == nstrips - 1)
    print(f"edge-strip runs: median {np.median(dur[edge]):.1f} us; interior: {np.median(dur[~edge]):.1f} us")
    for r in sorted(set(rows)):
        m = rows == r
        print(f"band {r} rows: {m.sum()} runs, median {np.median(dur[m]):.1f} us, max {dur[m].max():.1f}")
    smend = {}
    for k in range(len(sm)):
        smend[int(sm[k])] = max(smend.get(int(sm[k]), 0), end[k])
    v = np.array(sorted(smend.values()))
    print(f"SM finish times: min {v.min():.1f} median {np.median(v):.1f} max {v.max():.1f} us")
    slow = sorted(range(len(dur)), key=lambda k: -end[k])[:12]
    for k in slow:
        print(f"  last: end {end[k]:.1f} dur {dur[k]:.1f} start {start[k]:.1f} sm {int(sm[k])} strip {strip[k]} rows {rows[k]}")


if __name__ == "__main__":
    main()
