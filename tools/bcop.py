#!/usr/bin/env python
"""One call of one operator at the cfg3 shape (8 x 2048^2, CDF 9/7 / db4 periodic, 5 levels) after a warm-up,
for ncu launch lists:  python tools/bcop.py symmetric_edag adjoint"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_02018_b200 import wl  # noqa: E402

bc, op = sys.argv[1], sys.argv[2]
plan = wl.Plan(2048, 2048, 5, "cdf97" if bc != "periodic" else "db4", bc, "float32")
B = 8
img = torch.randn(B, 2048, 2048, device="cuda")
x = torch.randn(B, plan.p_alloc, device="cuda")
ox, oi = torch.empty_like(x), torch.empty_like(img)
fn = {"adjoint": lambda: plan.adjoint(img, out=ox), "synthesize": lambda: plan.synthesize(x, out=oi),
      "analyze": lambda: plan.analyze(img, out=ox)}[op]
for _ in range(3):
    fn()
torch.cuda.synchronize()
fn()
torch.cuda.synchronize()
