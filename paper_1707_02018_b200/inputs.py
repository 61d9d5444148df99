"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic (no filtering, extension or blur):
only the workload configurations of BASELINE.json and random draws.  Both the CUDA
path and the oracle consume what it returns; where a workload needs a blurred image
(config 5: b = R(blobs) + noise) the caller applies its own R.

Recipe:
  numpy Generator(PCG64(seed)), seed = 1000*cfg + s with s = 1: x, 2: y, 3: blobs, 4: noise;
  drawn in fp64 in the order stated, C order over [B, ...], then cast to the config dtype.
  x  : Bernoulli(rho) * N(0, 1) on the p_valid coefficients (packed order), or N(0,1) (cfg1)
  y  : N(0, 1) or U[0, 1) images
  blobs: 64 isotropic Gaussians per image; per blob cy ~ U[0,h), cx ~ U[0,w), sigma ~ U[8,128),
       a ~ U[0,1); image = sum_i a_i exp(-((r-cy_i)^2 + (c-cx_i)^2) / (2 sigma_i^2))
  noise: N(0, 1) scaled by 1e-3 (reading R13: "N(0,1e-3)" is the standard deviation)
The paper's own image (a resolution chart), PSF and noise are unpublished;
these synthetic inputs stand in for them.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    idx: int
    name: str
    h: int
    w: int
    batch: int
    filt: str
    bc: str
    levels: int
    dtype: str          # "float32" | "float64"
    x_density: float    # 1.0 = dense N(0,1)
    y_dist: str         # "normal" | "uniform"
    ops: tuple


CONFIGS = {
    1: Config(1, "cfg1_64_db2_per_f64", 64, 64, 1, "db2", "periodic", 3, "float64", 1.0, "normal", ("W", "W*")),
    2: Config(2, "cfg2_512_db4_sym", 512, 512, 1, "db4", "symmetric", 4, "float32", 0.05, "uniform",
              ("W", "W*", "Wdag")),
    3: Config(3, "cfg3_8x2048_cdf97_sym", 2048, 2048, 8, "cdf97", "symmetric", 5, "float32", 0.05, "normal",
              ("W", "W*")),
    4: Config(4, "cfg4_4096_db8_zero", 4096, 4096, 1, "db8", "zero", 6, "float32", 0.02, "normal", ("W", "W*")),
    5: Config(5, "cfg5_4x4096_cdf97_sym_grad", 4096, 4096, 4, "cdf97", "symmetric", 5, "float32", 0.05, "normal",
              ("grad",)),
}

BLUR_NTAPS, BLUR_SIGMA = 15, 3.0
NOISE_STD = 1e-3
N_BLOBS = 64


def rng(cfg_idx: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(1000 * cfg_idx + stream))


def coefficients(g: np.random.Generator, batch: int, p_valid: int, density: float) -> np.ndarray:
    """[batch, p_valid] fp64: Bernoulli(density) mask times N(0,1) (density 1: plain N(0,1))."""
    if density >= 1.0:
        return g.standard_normal((batch, p_valid))
    mask = g.random((batch, p_valid)) < density
    vals = g.standard_normal((batch, p_valid))
    return np.where(mask, vals, 0.0)


def images(g: np.random.Generator, batch: int, h: int, w: int, dist: str) -> np.ndarray:
    if dist == "uniform":
        return g.random((batch, h, w))
    return g.standard_normal((batch, h, w))


def blobs(g: np.random.Generator, batch: int, h: int, w: int, n: int = N_BLOBS) -> np.ndarray:
    """Smooth random images: sum of n Gaussian blobs per image (fp64 [batch, h, w])."""
    out = np.empty((batch, h, w))
    rr = np.arange(h, dtype=np.float64)
    cc = np.arange(w, dtype=np.float64)
    for b in range(batch):
        cy = np.empty(n); cx = np.empty(n); sg = np.empty(n); am = np.empty(n)
        for i in range(n):                      # per blob, in the order cy, cx, sigma, a
            cy[i] = g.uniform(0.0, h)
            cx[i] = g.uniform(0.0, w)
            sg[i] = g.uniform(8.0, 128.0)
            am[i] = g.uniform(0.0, 1.0)
        Gr = np.exp(-((rr[None, :] - cy[:, None]) ** 2) / (2.0 * sg[:, None] ** 2))     # [n, h]
        Gc = np.exp(-((cc[None, :] - cx[:, None]) ** 2) / (2.0 * sg[:, None] ** 2))     # [n, w]
        out[b] = (Gr.T * am[None, :]) @ Gc
    return out


def chart(h: int, w: int) -> np.ndarray:
    """Synthetic resolution-chart stand-in for the Weber 1993 test chart of P:104-110 (the chart
    itself is not in this container): fp64 [h, w] in [0, 1], background 0.  Groups of vertical and
    horizontal bar triplets with periods 2..32 px, four disks of decreasing radius and a grey ramp."""
    img = np.zeros((h, w))
    periods = [32, 24, 16, 12, 8, 6, 4, 3, 2]
    gx = w // (len(periods) + 1)
    for i, per in enumerate(periods):               # vertical bars, top band
        x0 = gx // 2 + i * gx
        for k in range(3):
            a = x0 + 2 * k * (per // 2 if per > 2 else 1)
            img[h // 16: h // 3, a: a + max(per // 2, 1)] = 1.0
    gy = h // (len(periods) + 1)
    for i, per in enumerate(periods):               # horizontal bars, left band of the lower half
        y0 = h // 3 + gy // 4 + i * (2 * h // 3) // (len(periods) + 1)
        for k in range(3):
            a = y0 + 2 * k * (per // 2 if per > 2 else 1)
            img[a: a + max(per // 2, 1), w // 16: w // 3] = 1.0
    yy, xx = np.mgrid[0:h, 0:w]
    for i, r in enumerate([h / 8, h / 12, h / 20, h / 40]):   # disks
        cy, cx = h / 2 + (i // 2) * h / 4, w / 2 + (i % 2) * w / 4
        img[(yy - cy) ** 2 + (xx - cx) ** 2 <= r * r] = 0.75
    img[h - h // 10:, w // 2:] = np.linspace(0.0, 1.0, w - w // 2)[None, :]  # ramp
    return img


# Example 2: two channels, true lengths K = 894, N = 1717, guessed K_est = 844, N_est = 1767,
# noise std 0.005; lambda_TV = 0.01, delta = 0.1.  The Rideout simulation is missing: spike trains stand in.
BCE = dict(channels=2, K=894, N=1717, K_est=844, N_est=1767, noise=0.005, lam_tv=0.01, delta=0.1)


def spikes(g: np.random.Generator, shape, density: float) -> np.ndarray:
    """Sparse spike train(s): Bernoulli(density) support x N(0, 1) amplitudes (fp64)."""
    mask = g.random(shape) < density
    return np.where(mask, g.standard_normal(shape), 0.0)


def bce_problem(seed: int, problems: int, channels: int, K: int, N: int, K_est: int, N_est: int,
                noise_std: float, density: float = 0.02):
    """One observed multi-channel record and `problems` random starts (the paper initialises h_i
    and s with N(0, 1) numbers).  Draw order: true h [C, K], true s [N], noise [C, K+N-1],
    then h0 [P, C, K_est], s0 [P, N_est].  Returns fp64 (h_true, s_true, noise, h0, s0); the observation
    x = h_true * s_true + noise is formed by the caller's own convolution."""
    assert K + N == K_est + N_est, "the guessed lengths must keep the observed length K+N-1"
    g = np.random.Generator(np.random.PCG64(seed))
    h_true = spikes(g, (channels, K), density)
    s_true = spikes(g, (N,), density)
    nz = noise_std * g.standard_normal((channels, K + N - 1))
    h0 = g.standard_normal((problems, channels, K_est))
    s0 = g.standard_normal((problems, N_est))
    return h_true, s_true, nz, h0, s0


def noise(g: np.random.Generator, batch: int, h: int, w: int) -> np.ndarray:
    return NOISE_STD * g.standard_normal((batch, h, w))


def workload(cfg: Config, p_valid: int, batch: int | None = None):
    """Draw (x_packed, y, blobs, noise) for a config in fp64 (blobs/noise only for cfg5)."""
    B = cfg.batch if batch is None else batch
    x = coefficients(rng(cfg.idx, 1), B, p_valid, cfg.x_density)
    y = images(rng(cfg.idx, 2), B, cfg.h, cfg.w, cfg.y_dist)
    bl = nz = None
    if cfg.idx == 5:
        bl = blobs(rng(cfg.idx, 3), B, cfg.h, cfg.w)
        nz = noise(rng(cfg.idx, 4), B, cfg.h, cfg.w)
    return x, y, bl, nz


def cast(a: np.ndarray, dtype: str) -> np.ndarray:
    """Round to the config dtype and back to fp64 (the oracle consumes exactly these values)."""
    return a.astype(np.float32).astype(np.float64) if dtype == "float32" else a.astype(np.float64)
