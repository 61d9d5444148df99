#!/usr/bin/env python
"""Benchmark of the hot path of arXiv 1707.02018 on B200: grad f = W* R* (R W x - b).

One step = one wl_grad call on BASELINE.json config 5 (4 x 4096^2 fp32, CDF 9/7, 5 levels,
symmetric BC, 15-tap sigma=3 Gaussian PSF); it runs every hot-path row (W, R, R*, W*).
Metric (BASELINE.json): "W* and grad f GB/s and % HBM roofline at 4096^2 fp32; gradient
evals/sec".  value = grad f GB/s = algorithmic bytes of the step (the sum of its operators'
minimum bytes) / device time.  W* at config 4 (4096^2 db8, 6 levels,
zero BC) is reported beside it under "wstar_cfg4".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl wl|reference]

N > 1 (torchrun): every rank runs the full config-5 batch on its own GPU (replicas, weak
scaling, no data-path collective -- DESIGN.md "Multi-GPU"); time = max over ranks.
--impl reference times the fp64 CPU oracle (the only other place bench.py runs oracle/).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import shutil
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "W* and ∇f GB/s and % HBM roofline at 4096² fp32; gradient evals/sec"
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback if MEASURED_PEAKS.json is absent
FFMA_PEAK_TFLOPS = 74.4     # 148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz (ALU ceiling)


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def grad_bytes(B, N, p, es):
    """Sum of the operators' minimum bytes: W (N+p) + [R u - b] (3N) + R* (2N) + W* (N+p)."""
    return es * B * ((N + p) + 3 * N + 2 * N + (N + p))


def traffic_from_profiles(kernel_key):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    v = d.get(kernel_key)
    return None if v is None else float(v)


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed region runs."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x2: "applications_clocks_setting", 0x80: "hw_power_brake_slowdown",
               0x1: "gpu_idle", 0x100: "sync_boost", 0x200: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self._stop = [], set(), threading.Event()
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - GPU box only
            self.err = str(e)

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup():
    """One process per GPU (torchrun env); the process group only brackets the timed region."""
    import torch

    from paper_1707_02018_b200 import replicas
    info = replicas.rank_info()
    if info.world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(info.local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", info.local))
    else:
        torch.cuda.set_device(0)
    return info.world, info.rank, info.local


def barrier(ws):
    from paper_1707_02018_b200 import replicas
    replicas.barrier(ws)


def max_over_ranks(v, ws):
    from paper_1707_02018_b200 import replicas
    return replicas.max_over_ranks(v, ws)


def time_calls(torch, fn, reps, warmup=3):
    """Average device ms per call on the current stream (events on the launching stream)."""
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def time_dist(torch, fn, reps, flush=None, warmup=3):
    """Per-call device time distribution (CUDA events on the launching stream):
    median / p10 / p90 ms over `reps` calls.  flush: a buffer of >= 2x the L2 size zeroed before
    every call, outside the events (cold L2); None: back-to-back calls (warm L2)."""
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        if flush is not None:
            flush.zero_()
        a.record(s)
        fn()
        b.record(s)
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) for a, b in ev])
    return {"median_ms": float(np.median(t)), "p10_ms": float(np.percentile(t, 10)),
            "p90_ms": float(np.percentile(t, 90)), "reps": int(reps),
            "l2": "cold (2x L2 memset before each call)" if flush is not None else "warm (back to back)"}


def l2_flush_buffer(torch, dev):
    """A scratch buffer of 2x the device's L2 (SURVEY §8(d) cold-L2 protocol)."""
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    return torch.empty(2 * l2 // 4 + 1024, dtype=torch.float32, device=dev), l2


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


_ONE_THREAD = r"""
import sys, time
sys.path.insert(0, {root!r})
from oracle import oracle as O
from paper_1707_02018_b200 import inputs
c = inputs.CONFIGS[5]
lay = O.layout(c.h, c.w, c.levels, c.filt, c.bc)
x, _, bl, nz = inputs.workload(c, lay.p, batch=1)
x = inputs.cast(x, c.dtype)
b = inputs.cast(O.blur(bl) + nz, c.dtype)
t = time.perf_counter()
O.grad(x, b, c.levels, c.filt, c.bc)
print(time.perf_counter() - t)
"""


def cpu_oracle_one_thread(timeout=240):
    """The fp64 oracle's cfg5 gradient on one 4096^2 image, pinned to one core with one OpenMP
    thread (taskset + OMP_NUM_THREADS=1); seconds, or None if it cannot run."""
    cpu = sorted(os.sched_getaffinity(0))[0]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-c", _ONE_THREAD.format(root=ROOT)]
    if shutil.which("taskset"):
        cmd = ["taskset", "-c", str(cpu)] + cmd
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=timeout)
        return float(out.stdout.strip().splitlines()[-1])
    except Exception:
        return None


# ------------------------------------------------------------------- oracle arm
def cpu_oracle_grad_step(c, plan_p_valid, x, b):
    from oracle import oracle as O
    t = time.perf_counter()
    O.grad(x, b, c.levels, c.filt, c.bc)
    return time.perf_counter() - t


def run_reference(args):
    """--impl reference: the fp64 CPU oracle as it stands, on the host cores (rank 0 only)."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_1707_02018_b200 import inputs
    c = inputs.CONFIGS[5]
    lay = O.layout(c.h, c.w, c.levels, c.filt, c.bc)
    # bounded sample: one of the four images of the config-5 batch per step
    x, _, bl, nz = inputs.workload(c, lay.p, batch=1)
    x = inputs.cast(x, c.dtype)
    b = inputs.cast(O.blur(bl) + nz, c.dtype)
    for _ in range(args.warmup):
        cpu_oracle_grad_step(c, lay.p, x, b)
    t = 0.0
    for _ in range(args.steps):
        t += cpu_oracle_grad_step(c, lay.p, x, b)
    step_s = t / args.steps
    nbytes = grad_bytes(1, c.h * c.w, lay.p, 4)
    val = nbytes / step_s / 1e9
    cores = len(os.sched_getaffinity(0))
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg5 grad f, 1 of 4 images per step (bounded sample)", "h": c.h, "w": c.w,
                       "batch": 1, "filter": c.filt, "bc": c.bc, "levels": c.levels},
            "cpu_baseline": {"value": val, "unit": "GB/s", "cores": cores, "kind": "oracle",
                             "sample": "1 image of 4096^2 per step (cfg5 has 4)", "cpu_model": cpu_model()},
            "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "grad_evals_per_s": 1.0 / step_s}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------- GPU arm
def run_wl(args):
    import torch

    from paper_1707_02018_b200 import inputs, wl

    ws, rank, local = dist_setup()
    dev = torch.device("cuda", local)
    hbm_peak, peak_src = measured_peaks()
    c = inputs.CONFIGS[5]
    plan = wl.Plan(c.h, c.w, c.levels, c.filt, c.bc, c.dtype)
    blur = wl.Blur(c.h, c.w, inputs.BLUR_NTAPS, inputs.BLUR_SIGMA, dtype=c.dtype)
    B, N, es = c.batch, c.h * c.w, 4
    # ---- inputs (untimed): x from the seeded generator; b = R(blobs) + noise with the GPU R
    xp, _, bl, nz = inputs.workload(c, plan.p_valid)
    x = torch.from_numpy(plan.from_packed(xp.astype(np.float32))).to(dev)
    blobs_d = torch.from_numpy(bl.astype(np.float32)).to(dev)
    b = blur.apply(blobs_d) + torch.from_numpy(nz.astype(np.float32)).to(dev)
    del blobs_d
    g = torch.empty_like(x)
    f = torch.zeros(B, dtype=torch.float64, device=dev)
    wsb = plan._ws(wl.OP_GRAD, B, blur=blur)
    step_eager = lambda: wl.grad(plan, blur, x, b, out=g, f=f, ws=wsb)  # noqa: E731
    # the step runs as a CUDA graph of the library's launches (one graph launch per step; the
    # same kernels, arguments and work as the eager call) unless --eager
    graph = None if args.eager else wl.Graph(step_eager)
    step = step_eager if graph is None else graph.replay
    per_step = (graph.launches if graph is not None else None)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = wl.launch_count()
    with ClockSampler(local) as clk:
        e0.record(s)
        for _ in range(args.steps):
            step()
        e1.record(s)
        torch.cuda.synchronize()
    launches = wl.launch_count() - launches0 if graph is None else per_step * args.steps
    barrier(ws)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, ws)
    ms_eager = ms if graph is None else max_over_ranks(time_calls(torch, step_eager, max(args.steps, 5)), ws)
    nbytes = grad_bytes(B, N, plan.p_valid, es)
    value = ws * nbytes / (ms * 1e-3) / 1e9
    # per-step distributions beside the contract loop: cold L2 (primary) and warm
    flush, l2_bytes = l2_flush_buffer(torch, dev)
    dist_reps = max(args.steps, 20)
    step_dist = {"cold": time_dist(torch, step, dist_reps, flush), "warm": time_dist(torch, step, dist_reps)}
    step_dist["cold"]["GB/s"] = nbytes / (step_dist["cold"]["median_ms"] * 1e-3) / 1e9

    # ---- per-kernel live timing (events on the launching stream) for the roofline object
    u = torch.empty(B, c.h, c.w, device=dev)
    sres = torch.empty_like(u)
    plan.synthesize(x, out=u)
    reps = max(args.steps, 10)
    kernels = {}
    t_res = time_calls(torch, lambda: blur.residual_adjoint(u, b, out=sres), reps)
    # FLOPs: 4 separable 15-tap passes = 60 MAC per pixel (algorithmic, halo frame excluded)
    kernels["blur_residual_adjoint"] = {"ms": t_res, "bytes": 3 * N * es * B, "flops": 2.0 * 60 * N * B}
    p1 = wl.Plan(c.h, c.w, 1, c.filt, c.bc, c.dtype)
    x1 = torch.empty(B, p1.p_alloc, device=dev)
    t_a1 = time_calls(torch, lambda: p1.adjoint(u, out=x1), reps)
    kernels["analysis_level1_Wstar"] = {"ms": t_a1, "bytes": es * B * (N + p1.p_valid)}
    t_s1 = time_calls(torch, lambda: p1.synthesize(x1, out=u), reps)
    kernels["synthesis_level1_W"] = {"ms": t_s1, "bytes": es * B * (N + p1.p_valid)}
    # the same kernels with the cold-L2 protocol (median, p10 / p90)
    cold = {"blur_residual_adjoint": time_dist(torch, lambda: blur.residual_adjoint(u, b, out=sres), reps, flush),
            "analysis_level1_Wstar": time_dist(torch, lambda: p1.adjoint(u, out=x1), reps, flush),
            "synthesis_level1_W": time_dist(torch, lambda: p1.synthesize(x1, out=u), reps, flush)}
    for name, d in cold.items():
        kernels[name]["cold"] = d
        kernels[name]["cold"]["GB/s"] = kernels[name]["bytes"] / (d["median_ms"] * 1e-3) / 1e9
    for k in kernels.values():
        k["GB/s"] = k["bytes"] / (k["ms"] * 1e-3) / 1e9
        k["frac"] = k["GB/s"] / hbm_peak
        k["share_of_step"] = k["ms"] / ms
        if "flops" in k:  # the same kernel against the FP32 FMA ceiling (it sits near the ridge)
            k["TFLOP/s"] = k["flops"] / (k["ms"] * 1e-3) / 1e12
            k["alu_frac"] = k["TFLOP/s"] / FFMA_PEAK_TFLOPS
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    dk = kernels[dom]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": dk["GB/s"], "peak": hbm_peak, "unit": "GB/s",
                "frac": dk["frac"], "traffic": traffic_from_profiles(dom), "peak_source": peak_src,
                "bytes_per_launch": dk["bytes"]}

    # ---- W* at config 4 (the metric's other half)
    c4 = inputs.CONFIGS[4]
    plan4 = wl.Plan(c4.h, c4.w, c4.levels, c4.filt, c4.bc, c4.dtype)
    _, y4, _, _ = inputs.workload(c4, plan4.p_valid)
    y4 = torch.from_numpy(y4.astype(np.float32)).to(dev)
    x4 = torch.empty(1, plan4.p_alloc, device=dev)
    ws4 = plan4._ws(wl.OP_ADJOINT, 1)
    g4 = wl.Graph(lambda: plan4.adjoint(y4, out=x4, ws=ws4))
    b4 = 4 * (c4.h * c4.w + plan4.p_valid)
    d4c = time_dist(torch, g4.replay, max(args.steps, 30), flush)       # primary: cold L2
    d4w = time_dist(torch, g4.replay, max(args.steps, 30))              # beside it: warm
    t4 = d4c["median_ms"]
    t4e = time_dist(torch, lambda: plan4.adjoint(y4, out=x4, ws=ws4), max(args.steps, 30), flush)
    wstar = {"us": t4 * 1e3, "GB/s": b4 / (t4 * 1e-3) / 1e9, "frac": b4 / (t4 * 1e-3) / 1e9 / hbm_peak,
             "bytes": b4, "config": "cfg4 4096^2 db8 zero 6 levels fp32", "launch": "cuda_graph",
             "l2": "cold (2x L2 memset before each call); warm beside it", "cold": d4c, "warm": d4w,
             "warm_us": d4w["median_ms"] * 1e3, "eager_cold_us": t4e["median_ms"] * 1e3,
             "traffic": traffic_from_profiles("wstar_cfg4_chain")}
    del y4, x4, ws4

    # ---- the same gradient with the paper-literal symmetric adjoint (bc = symmetric_edag, reading R1
    # "P": W*_P = W~dagger_zpd (E_sym^dagger)*, Eq. (4)), the variant the paper's Fig. 2-3 runs
    plan_e = wl.Plan(c.h, c.w, c.levels, c.filt, "symmetric_edag", c.dtype)
    xe = plan_e.from_packed(plan.to_packed(x))
    ge = torch.empty_like(xe)
    wse = plan_e._ws(wl.OP_GRAD, B, blur=blur)
    de = time_dist(torch, wl.Graph(lambda: wl.grad(plan_e, blur, xe, b, out=ge, ws=wse)).replay, max(args.steps, 20), flush)
    grad_edag = {"ms": de["median_ms"], "GB/s": grad_bytes(B, N, plan_e.p_valid, es) / (de["median_ms"] * 1e-3) / 1e9,
                 "cold": de, "config": "cfg5 with bc=symmetric_edag", "launch": "cuda_graph"}
    del xe, ge, wse

    # ---- one FISTA iteration at cfg5 (grad f(y) + fused prox/momentum update)
    xf, yf = torch.zeros_like(x), x.clone()
    wsf = plan._ws(wl.OP_FISTA, B, blur=blur)
    t_dev = torch.full((1,), 2.0, dtype=torch.float64, device=dev)
    f_step = lambda: wl.fista_step(plan, blur, b, xf, yf, t_dev, 1e-3, 1.0, ws=wsf)  # noqa: E731
    tf_eager = time_calls(torch, f_step, reps)
    tf = time_calls(torch, wl.Graph(f_step).replay, reps)
    fista = {"ms_per_iter": tf, "iters_per_s": ws / (tf * 1e-3), "update_overhead_ms": tf - ms,
             "ms_per_iter_eager": tf_eager, "launch": "cuda_graph (device-resident t)",
             "config": "cfg5, lambda 1e-3, L 1"}
    del xf, yf, wsf

    # ---- W, W*, W-dagger at every other BASELINE config ("W and W-dagger rows for every
    # config"), graph-replayed, algorithmic bytes es*B*(N + p) per operator
    per_cfg = {}
    for ci in (1, 2, 3, 4):
        cc = inputs.CONFIGS[ci]
        pc = wl.Plan(cc.h, cc.w, cc.levels, cc.filt, cc.bc, cc.dtype)
        td = pc.torch_dtype
        gen = torch.Generator(dev).manual_seed(ci)
        imc = torch.randn(cc.batch, cc.h, cc.w, device=dev, dtype=td, generator=gen)
        xc = pc.from_packed(torch.randn(cc.batch, pc.p_valid, device=dev, dtype=td, generator=gen))
        oxc, oic = torch.empty_like(xc), torch.empty_like(imc)
        wss = {op: pc._ws(op, cc.batch) for op in (wl.OP_SYNTHESIZE, wl.OP_ADJOINT, wl.OP_ANALYZE)}
        nb = td.itemsize * cc.batch * (cc.h * cc.w + pc.p_valid)
        row = {"config": f"{cc.batch}x{cc.h}x{cc.w} {cc.filt} {cc.bc} J={cc.levels} {cc.dtype}", "bytes": nb}
        for name, fn in (("W", lambda: pc.synthesize(xc, out=oic, ws=wss[wl.OP_SYNTHESIZE])),
                         ("W*", lambda: pc.adjoint(imc, out=oxc, ws=wss[wl.OP_ADJOINT])),
                         ("W-dagger", lambda: pc.analyze(imc, out=oxc, ws=wss[wl.OP_ANALYZE]))):
            tt = time_calls(torch, wl.Graph(fn).replay, 20)
            row[name] = {"us": tt * 1e3, "GB/s": nb / (tt * 1e-3) / 1e9, "frac": nb / (tt * 1e-3) / 1e9 / hbm_peak}
        per_cfg[f"cfg{ci}"] = row
        del imc, xc, oxc, oic, wss

    # ---- Example 2: fused Eq. (6) gradient, paper sizes, 4096 random starts
    bc = inputs.BCE
    P_bce, C_b, K_b, N_b = 4096, bc["channels"], bc["K_est"], bc["N_est"]
    _, _, _, h0, s0 = inputs.bce_problem(7, P_bce, C_b, bc["K"], bc["N"], K_b, N_b, bc["noise"])
    hb_ = torch.from_numpy(h0.astype(np.float32)).to(dev)
    sb_ = torch.from_numpy(s0.astype(np.float32)).to(dev)
    xb_ = torch.randn(C_b, K_b + N_b - 1, device=dev, generator=torch.Generator(dev).manual_seed(7))
    ghb, gsb = torch.empty_like(hb_), torch.empty_like(sb_)
    fb_ = torch.empty(P_bce, dtype=torch.float64, device=dev)
    t_b = time_calls(torch, lambda: wl.bce_grad(hb_, sb_, xb_, bc["lam_tv"], bc["delta"], gh=ghb, gs=gsb, f=fb_),
                     max(args.steps, 10))
    flops_b = 2.0 * 3 * C_b * K_b * N_b * P_bce
    tf_b = flops_b / (t_b * 1e-3) / 1e12
    bce = {"workload": f"Eq. (6) gradient, {P_bce} random starts x {C_b} channels, K={K_b}, N={N_b}, fp32",
           "ms": t_b, "grads_per_s": ws * P_bce / (t_b * 1e-3),
           "roofline": {"bound": "alu", "achieved": tf_b, "peak": FFMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                        "frac": tf_b / FFMA_PEAK_TFLOPS, "flops_per_launch": flops_b,
                        "peak_source": "148 SMs x 128 FP32 lanes x 2 x 1.965 GHz (DESIGN.md §6)"}}
    del hb_, sb_, xb_, ghb, gsb, fb_

    # ---- end to end through the public API with host buffers (pinned), copies inside
    xh = x.cpu().pin_memory()
    bh = b.cpu().pin_memory()
    gh = torch.empty_like(xh).pin_memory()
    fh = torch.empty(B, dtype=torch.float64).pin_memory()

    wsh = plan._ws(wl.OP_GRAD_HOST, B, blur=blur)

    def e2e_step():  # the public host-buffer call: copies in, gradient, copies out, pipelined per image
        wl.grad_host(plan, blur, xh, bh, out=gh, f=fh, ws=wsh)

    e2e_steps = max(3, min(args.steps, 10))
    t_e2e = max_over_ranks(time_calls(torch, e2e_step, e2e_steps, warmup=2), ws)
    e2e = {"value": ws * nbytes / (t_e2e * 1e-3) / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": (xh.numel() + bh.numel()) * 4, "d2h_bytes_per_step": gh.numel() * 4 + B * 8,
           "ms_per_step": t_e2e}

    # ---- CPU oracle baseline (rank 0, N = 1 only, bounded sample)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        x1h, _, bl1, nz1 = inputs.workload(c, plan.p_valid, batch=1)
        x1h = inputs.cast(x1h, c.dtype)
        b1 = inputs.cast(O.blur(bl1) + nz1, c.dtype)
        reps_cpu = 3
        ts = sorted(cpu_oracle_grad_step(c, plan.p_valid, x1h, b1) for _ in range(reps_cpu))
        t = ts[len(ts) // 2]
        nb1 = grad_bytes(1, N, plan.p_valid, es)
        t1 = None if args.no_single_thread else cpu_oracle_one_thread()
        cpu = {"value": nb1 / t / 1e9, "unit": "GB/s", "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
               "sample": f"1 of the 4 cfg5 images (4096^2) per timing, median of {reps_cpu}, all host cores (OpenMP)",
               "s_per_image": t, "cpu_model": cpu_model(),
               "single_thread": None if t1 is None else {
                   "value": nb1 / t1 / 1e9, "unit": "GB/s", "cores": 1, "s_per_image": t1,
                   "sample": "1 cfg5 image, taskset to one core, OMP_NUM_THREADS=1, one timing"}}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": "cfg5: grad f = W* R* (R W x - b), 4 x 4096^2, CDF 9/7, 5 levels, "
                                       "symmetric BC, 15-tap sigma 3 Gaussian PSF",
                           "global_batch": B * ws, "h": c.h, "w": c.w, "levels": c.levels, "filter": c.filt,
                           "bc": c.bc, "parallelism": f"replicas x{ws}",
                           "l2": "inputs larger than L2 (x + b = 538 MB per step per GPU), no flush",
                           "launch": "each step = one replay of a CUDA graph of the wl_grad launches (--eager: direct calls)",
                           "bytes_per_step_per_gpu": nbytes},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary(), "step_launch": "eager" if graph is None else "cuda_graph",
                "ms_per_step_eager": ms_eager, "step_distribution": step_dist, "l2_bytes": l2_bytes, "grad_evals_per_s": ws / (ms * 1e-3), "images_per_s": ws * B / (ms * 1e-3),
                "grad_frac_of_hbm_roofline": value / ws / hbm_peak, "wstar_cfg4": wstar, "grad_cfg5_symmetric_edag": grad_edag, "fista_cfg5": fista, "bce": bce, "operators_by_config": per_cfg, "kernels": kernels}
        print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="wl", choices=["wl", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-single-thread", action="store_true", help="skip the one-core oracle timing")
    ap.add_argument("--eager", action="store_true", help="launch the timed step eagerly instead of as a CUDA graph")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_wl(args)


if __name__ == "__main__":
    sys.exit(main())
