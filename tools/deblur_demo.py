"""Deblurring with on-device FISTA: the analogue of the paper's Figs. 2-3 experiment (P:104-121,
P:172-180) on a synthetic resolution chart (inputs.chart; the Weber chart is not available).

For each wavelet (3-stage Haar and CDF 9/7, symmetric BC, as P:117 and P:174; both readings of
the symmetric W: the crop pair `symmetric` and the paper-literal `symmetric_edag`) and each closing
operator (true adjoint W* vs the approximation W-dagger), runs `--iters` FISTA iterations with
lambda = 2e-5 on b = R(chart) + noise and reports the relative error of W x against the
chart, the fraction of nonzero coefficients and an SSIM trace (Wang 2004 with the usual defaults:
11x11 Gaussian window sigma 1.5, k1 0.01, k2 0.03, dynamic range 1).  Every iteration runs in
libwl (one eager iteration, then a CUDA graph of one iteration with the momentum scalar t kept on
the device, replayed); only the metrics are computed on the host from copies taken every
`--every` iterations (the timer excludes them).

    python tools/deblur_demo.py --size 512 --iters 2500 --out profiles/r01_deblur_demo.json
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def ssim(a, b, sigma=1.5, k1=0.01, k2=0.03, L=1.0):
    from scipy.ndimage import gaussian_filter
    f = lambda z: gaussian_filter(z, sigma, truncate=3.5, mode="reflect")  # noqa: E731  (radius 5: 11x11)
    c1, c2 = (k1 * L) ** 2, (k2 * L) ** 2
    ma, mb = f(a), f(b)
    saa, sbb, sab = f(a * a) - ma * ma, f(b * b) - mb * mb, f(a * b) - ma * mb
    m = ((2 * ma * mb + c1) * (2 * sab + c2)) / ((ma * ma + mb * mb + c1) * (saa + sbb + c2))
    return float(m.mean())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--iters", type=int, default=2500)
    ap.add_argument("--every", type=int, default=100)
    ap.add_argument("--lam", type=float, default=2e-5)
    ap.add_argument("--noise", type=float, default=1e-3)
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch

    from paper_1707_02018_b200 import inputs, wl

    n = args.size
    truth = inputs.chart(n, n)
    dev = torch.device("cuda")
    td = getattr(torch, args.dtype)
    blur = wl.Blur(n, n, inputs.BLUR_NTAPS, inputs.BLUR_SIGMA, dtype=args.dtype)
    b = blur.apply(torch.from_numpy(truth).to(dev, td)[None])
    b += torch.from_numpy(args.noise * np.random.default_rng(7).standard_normal((1, n, n))).to(dev, td)
    results = {"size": n, "iters": args.iters, "lambda": args.lam, "noise_std": args.noise, "levels": args.levels,
               "psf": f"{inputs.BLUR_NTAPS}-tap Gaussian sigma {inputs.BLUR_SIGMA}, symmetric BC",
               "dtype": args.dtype, "image": "inputs.chart (synthetic resolution chart)", "runs": []}
    for filt, bc in (("haar", "symmetric"), ("cdf97", "symmetric"), ("haar", "symmetric_edag"),
                     ("cdf97", "symmetric_edag")):
        plan = wl.Plan(n, n, args.levels, filt, bc, args.dtype)
        lip = wl.lipschitz(plan, blur, iters=100)
        for adjoint in ("true", "pinv"):
            x = torch.zeros(1, plan.p_alloc, device=dev, dtype=td)
            y = x.clone()
            ws = plan._ws(wl.OP_FISTA, 1, blur=blur)
            t_dev = torch.ones(1, dtype=torch.float64, device=dev)
            step = lambda: wl.fista_step(plan, blur, b, x, y, t_dev, args.lam, lip, ws=ws,  # noqa: E731
                                         adjoint=adjoint)
            step()                                   # iteration 1 (eager), then graph replays
            graph = wl.Graph(step, warmup=0)
            trace = []
            ms = 0.0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for k in range(2, args.iters + 1):
                graph.replay()
                if k % args.every == 0 or k == args.iters:
                    e1.record()
                    torch.cuda.synchronize()
                    ms += e0.elapsed_time(e1)
                    img = plan.synthesize(x)[0].double().cpu().numpy()
                    trace.append({"iter": k, "ssim": ssim(img, truth),
                                  "rel_err": float(np.linalg.norm(img - truth) / np.linalg.norm(truth))})
                    e0.record()
            xv = plan.to_packed(x.double().cpu().numpy())
            run = {"wavelet": filt, "bc": bc, "adjoint": "W*" if adjoint == "true" else "W-dagger", "lipschitz": lip,
                   "rel_err": trace[-1]["rel_err"], "nnz_fraction": float(np.mean(np.abs(xv) > 1e-12)),
                   "ssim": trace[-1]["ssim"], "trace": trace,
                   "ms_per_iter": ms / max(args.iters - 1, 1)}
            results["runs"].append(run)
            print(json.dumps({k: v for k, v in run.items() if k != "trace"}), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(results, fh, indent=1)


if __name__ == "__main__":
    main()
