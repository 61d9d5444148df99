#!/usr/bin/env python
"""Per-operator timing on one GPU (development tool; bench.py is the contract).

  python tools/opbench.py --cfg 4 --op adjoint --reps 50
ops: adjoint, analyze, analyze_adjoint, synthesize, blur, residual, grad, fista.  Prints one JSON line per op with
device ms per call (CUDA events, warm L2 for small configs).
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1707_02018_b200 import inputs, wl
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=4)
    ap.add_argument("--op", default="adjoint")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--levels", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    a = ap.parse_args()
    c = inputs.CONFIGS[a.cfg]
    J = a.levels or c.levels
    B = a.batch or c.batch
    plan = wl.Plan(c.h, c.w, J, c.filt, c.bc, c.dtype)
    dt = plan.torch_dtype
    img = torch.randn(B, c.h, c.w, device="cuda", dtype=dt)
    img2 = torch.randn(B, c.h, c.w, device="cuda", dtype=dt)
    x = torch.randn(B, plan.p_alloc, device="cuda", dtype=dt)
    out_x = torch.empty_like(x)
    out_i = torch.empty_like(img)
    blur = wl.Blur(c.h, c.w, 15, 3.0, dtype=c.dtype)
    ops = a.op.split(",")
    for op in ops:
        if op == "adjoint":
            ws = plan._ws(wl.OP_ADJOINT, B)
            fn = lambda: plan.adjoint(img, out=out_x, ws=ws)  # noqa: E731
            nbytes = (c.h * c.w + plan.p_valid) * B * plan.torch_dtype.itemsize
        elif op == "analyze":
            ws = plan._ws(wl.OP_ANALYZE, B)
            fn = lambda: plan.analyze(img, out=out_x, ws=ws)  # noqa: E731
            nbytes = (c.h * c.w + plan.p_valid) * B * plan.torch_dtype.itemsize
        elif op == "analyze_adjoint":
            ws = plan._ws(wl.OP_ANALYZE_ADJOINT, B)
            fn = lambda: plan.analyze_adjoint(x, out=out_i, ws=ws)  # noqa: E731
            nbytes = (c.h * c.w + plan.p_valid) * B * plan.torch_dtype.itemsize
        elif op == "synthesize":
            ws = plan._ws(wl.OP_SYNTHESIZE, B)
            fn = lambda: plan.synthesize(x, out=out_i, ws=ws)  # noqa: E731
            nbytes = (c.h * c.w + plan.p_valid) * B * plan.torch_dtype.itemsize
        elif op == "blur":
            fn = lambda: blur.apply(img, out=out_i)  # noqa: E731
            nbytes = 2 * c.h * c.w * B * plan.torch_dtype.itemsize
        elif op == "residual":
            fn = lambda: blur.residual_adjoint(img, img2, out=out_i)  # noqa: E731
            nbytes = 3 * c.h * c.w * B * plan.torch_dtype.itemsize
        elif op == "grad":
            ws = plan._ws(wl.OP_GRAD, B, blur=blur)
            fn = lambda: wl.grad(plan, blur, x, img2, out=out_x, ws=ws)  # noqa: E731
            nbytes = (6 * c.h * c.w + 2 * (c.h * c.w + plan.p_valid)) * B * plan.torch_dtype.itemsize
        elif op == "fista":
            ws = plan._ws(wl.OP_FISTA, B, blur=blur)
            xf, yf = torch.zeros_like(x), x.clone()
            t_dev = torch.full((1,), 2.0, dtype=torch.float64, device="cuda")
            fn = lambda: wl.fista_step(plan, blur, img2, xf, yf, t_dev, 1e-3, 1.0, ws=ws)  # noqa: E731
            nbytes = (6 * c.h * c.w + 2 * (c.h * c.w + plan.p_valid) + 3 * plan.p_valid) * B * plan.torch_dtype.itemsize
        else:
            raise SystemExit(f"unknown op {op}")
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(json.dumps({"cfg": a.cfg, "op": op, "levels": J, "batch": B, "us": ms * 1e3,
                          "GB/s": nbytes / (ms * 1e-3) / 1e9}))


if __name__ == "__main__":
    main()
