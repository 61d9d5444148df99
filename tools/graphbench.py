#!/usr/bin/env python
"""Eager vs CUDA-graph replay of whole operator calls (development tool).

  python tools/graphbench.py --cfg 5 --op grad --reps 30
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1707_02018_b200 import inputs, wl
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=5)
    ap.add_argument("--op", default="grad")
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    c = inputs.CONFIGS[a.cfg]
    plan = wl.Plan(c.h, c.w, c.levels, c.filt, c.bc, c.dtype)
    dt = plan.torch_dtype
    B = c.batch
    blur = wl.Blur(c.h, c.w, 15, 3.0, dtype=c.dtype)
    x = torch.randn(B, plan.p_alloc, device="cuda", dtype=dt)
    img = torch.randn(B, c.h, c.w, device="cuda", dtype=dt)
    out_x = torch.empty_like(x)
    out_i = torch.empty_like(img)
    if a.op == "grad":
        ws = plan._ws(wl.OP_GRAD, B, blur=blur)
        fn = lambda: wl.grad(plan, blur, x, img, out=out_x, ws=ws)  # noqa: E731
    elif a.op == "adjoint":
        ws = plan._ws(wl.OP_ADJOINT, B)
        fn = lambda: plan.adjoint(img, out=out_x, ws=ws)  # noqa: E731
    else:
        ws = plan._ws(wl.OP_SYNTHESIZE, B)
        fn = lambda: plan.synthesize(x, out=out_i, ws=ws)  # noqa: E731

    def timeit(f):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps * 1e3

    eager = timeit(fn)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    graph = timeit(g.replay)
    print(json.dumps({"cfg": a.cfg, "op": a.op, "eager_us": eager, "graph_us": graph}))


if __name__ == "__main__":
    main()
