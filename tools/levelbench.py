#!/usr/bin/env python
"""Marginal cost of each level of the W* / W / W-dagger chains (development tool).

  python tools/levelbench.py --cfg 4 --ops adjoint,synthesize
Times the whole chain for J = 1 .. levels (CUDA-graph replay, eager beside it, warm and cold L2) and prints one
JSON line per (op, J); the difference between consecutive J is the cost level J adds to the chain.
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
    ap.add_argument("--cfg", type=int, default=4)
    ap.add_argument("--ops", default="adjoint,synthesize")
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    c = inputs.CONFIGS[a.cfg]
    B = c.batch
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    flush = torch.empty(2 * l2, dtype=torch.uint8, device="cuda")
    for op in a.ops.split(","):
        for J in range(1, c.levels + 1):
            plan = wl.Plan(c.h, c.w, J, c.filt, c.bc, c.dtype)
            dt = plan.torch_dtype
            img = torch.randn(B, c.h, c.w, device="cuda", dtype=dt)
            x = torch.randn(B, plan.p_alloc, device="cuda", dtype=dt)
            out_x, out_i = torch.empty_like(x), torch.empty_like(img)
            opc = {"adjoint": wl.OP_ADJOINT, "analyze": wl.OP_ANALYZE, "synthesize": wl.OP_SYNTHESIZE}[op]
            ws = plan._ws(opc, B)
            if op == "adjoint":
                fn = lambda: plan.adjoint(img, out=out_x, ws=ws)  # noqa: E731
            elif op == "analyze":
                fn = lambda: plan.analyze(img, out=out_x, ws=ws)  # noqa: E731
            else:
                fn = lambda: plan.synthesize(x, out=out_i, ws=ws)  # noqa: E731
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                fn()
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()

            def timed(f, cold):
                ts = []
                for _ in range(a.reps):
                    if cold:
                        flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    f()
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e3)
                ts.sort()
                return ts[len(ts) // 2]

            print(json.dumps({"cfg": a.cfg, "op": op, "J": J, "graph_warm_us": timed(g.replay, False),
                              "graph_cold_us": timed(g.replay, True), "eager_cold_us": timed(fn, True),
                              "launches": None}), flush=True)


if __name__ == "__main__":
    main()
