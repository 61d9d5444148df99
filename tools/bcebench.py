#!/usr/bin/env python
"""Example 2 kernels on one GPU (development tool): the fused Eq. (6) gradient and the three
correlation operators at the paper's sizes (C = 2, K_est = 844, N_est = 1767), P random starts.

  python tools/bcebench.py --problems 4096 --reps 20 [--dtype float32]
Prints one JSON line per op: device ms per call, algorithmic TFLOP/s (2 flop per MAC of the
defining sums, zero padding excluded) and the fraction of the FP32 FFMA peak (74.4 TFLOP/s).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

FFMA_PEAK_TFLOPS = 74.4


def main():
    import torch

    from paper_1707_02018_b200 import wl
    ap = argparse.ArgumentParser()
    ap.add_argument("--problems", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--K", type=int, default=844)
    ap.add_argument("--N", type=int, default=1767)
    ap.add_argument("--C", type=int, default=2)
    a = ap.parse_args()
    dt = getattr(torch, a.dtype)
    P, C, K, N = a.problems, a.C, a.K, a.N
    M = K + N - 1
    h = torch.randn(P, C, K, device="cuda", dtype=dt)
    s = torch.randn(P, N, device="cuda", dtype=dt)
    x = torch.randn(C, M, device="cuda", dtype=dt)
    r = torch.randn(P * C, M, device="cuda", dtype=dt)
    hf, sf = h.reshape(P * C, K), s.repeat_interleave(C, 0)
    f = torch.zeros(P, dtype=torch.float64, device="cuda")
    gh, gs = torch.empty_like(h), torch.empty_like(s)
    ops = {
        "bce_grad": (lambda: wl.bce_grad(h, s, x, 0.01, 0.1, gh=gh, gs=gs, f=f), 3 * C * K * N * P),
        "conv_full": (lambda: wl.conv_full(hf, sf), C * K * N * P),
        "conv_adjoint_h": (lambda: wl.conv_adjoint_h(sf, r, K), C * K * N * P),
        "conv_adjoint_s": (lambda: wl.conv_adjoint_s(hf, r, N), C * K * N * P),
    }
    for name, (fn, macs) in ops.items():
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
        tf = 2 * macs / (ms * 1e-3) / 1e12
        print(json.dumps({"op": name, "problems": P, "C": C, "K": K, "N": N, "dtype": a.dtype, "ms": ms,
                          "TFLOP/s": tf, "frac_ffma_peak": tf / FFMA_PEAK_TFLOPS}), flush=True)


if __name__ == "__main__":
    main()
