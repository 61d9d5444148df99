#!/usr/bin/env python
"""W*, W, W-dagger under every boundary condition at the cfg3 shape (8 x 2048^2), CUDA-graph replay."""
import os, sys, torch, json
sys.path.insert(0, os.getcwd())
from paper_1707_02018_b200 import wl
for bc in ("symmetric", "symmetric_edag", "periodic", "zero"):
    plan = wl.Plan(2048, 2048, 5, "cdf97" if bc != "periodic" else "db4", bc, "float32")
    B = 8
    img = torch.randn(B, 2048, 2048, device="cuda"); x = torch.randn(B, plan.p_alloc, device="cuda")
    ox, oi = torch.empty_like(x), torch.empty_like(img)
    res = {"bc": bc}
    for name, fn in (("W*", lambda: plan.adjoint(img, out=ox)), ("W", lambda: plan.synthesize(x, out=oi)), ("Wdag", lambda: plan.analyze(img, out=ox))):
        g = wl.Graph(fn)
        for _ in range(3): g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): g.replay()
        e1.record(); torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
    print(json.dumps(res))
