#!/usr/bin/env python
"""Tiny W (synthesize) repro across filters / BCs / dtypes (debug helper; prints first failure)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1707_02018_b200 import wl
from oracle import oracle as O

cases = [(f, bc, dt, shp) for bc in sys.argv[1].split(",") for f in sys.argv[2].split(",")
         for dt in ("float64", "float32") for shp in ((37, 45, 2), (130, 97, 3))]
for f, bc, dt, (h, w, J) in cases:
    plan = wl.Plan(h, w, J, f, bc, dt)
    rng = np.random.default_rng(0)
    xp = rng.standard_normal((2, plan.p_valid))
    if dt == "float32":
        xp = xp.astype(np.float32).astype(np.float64)
    xd = torch.from_numpy(plan.from_packed(xp)).to("cuda", getattr(torch, dt))
    try:
        y = plan.synthesize(xd)
        torch.cuda.synchronize()
    except Exception as e:
        print("FAIL", f, bc, dt, h, w, J, repr(e)[:200]); sys.exit(1)
    ref = O.synthesize(xp, h, w, J, f, bc)
    err = np.linalg.norm(y.double().cpu().numpy() - ref) / np.linalg.norm(ref)
    print(f, bc, dt, h, w, J, f"{err:.2e}", flush=True)
