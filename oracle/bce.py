"""fp64 oracle for Example 2, blind channel estimation (PAPER.md §"Example 2: Blind Channel
Estimation").  TEST INFRASTRUCTURE ONLY: imported solely by `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / reference legs.

Every function is the paper's sum written out, one output index at a time (a dot product over
the summation index is the only library step), in the paper's notation:
  conv_full        x_est = h * s, the "full" zero-padded linear convolution, length K+N-1
                   x_est[m] = sum_k h[k] s[m-k]  (the matrices displayed at P:216-226)
  conv_adjoint_h   S* r:  grad_h[n] = sum_{k<N} s[k] r[k+n],  n < K   (the "valid"
                   cross-correlation of r with s; MATLAB conv(r, conj(s(end:-1:1)), 'valid'))
  conv_adjoint_s   H* r:  grad_s[k] = sum_{n<K} h[n] r[k+n],  k < N   ("very similar")
  huber            L_delta(z); tv_soft(h) = L_delta(D h) / delta with (D h)_j = h_{j+1} - h_j
  bce_smooth       the smooth part of Eq. (6) for C channels sharing s:
                   F = sum_i ( ||h_i * s - x_i||^2 + lam_tv L_delta(D h_i) / delta ),
                   literally as printed -- without the 1/2 of Eq. (5), hence the factor 2 in its
                   gradient (reading R24):
                   grad_{h_i} = 2 S* r_i + (lam_tv / delta) D^T psi(D h_i),
                   grad_s     = 2 sum_i H_i* r_i,      r_i = h_i * s - x_i,  psi = L_delta'.
Real signals only (the paper's experiment is real), so conj() is the identity.
"""
from __future__ import annotations

import numpy as np


def conv_full(h, s):
    """x_est[m] = sum_k h[k] s[m-k], m = 0 .. K+N-2 (zero-padded boundaries)."""
    h = np.asarray(h, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    K, N = h.shape[-1], s.shape[-1]
    out = np.zeros(np.broadcast_shapes(h.shape[:-1], s.shape[:-1]) + (K + N - 1,))
    for m in range(K + N - 1):
        k = np.arange(max(0, m - N + 1), min(K, m + 1))
        out[..., m] = np.sum(h[..., k] * s[..., m - k], axis=-1)
    return out


def conv_adjoint_h(s, r, K: int):
    """S* r: grad_h[n] = sum_{k<N} s[k] r[k+n] for n < K."""
    s = np.asarray(s, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    N = s.shape[-1]
    assert r.shape[-1] == K + N - 1
    out = np.zeros(np.broadcast_shapes(s.shape[:-1], r.shape[:-1]) + (K,))
    for n in range(K):
        out[..., n] = np.sum(s * r[..., n:n + N], axis=-1)
    return out


def conv_adjoint_s(h, r, N: int):
    """H* r: grad_s[k] = sum_{n<K} h[n] r[k+n] for k < N (the s-side analogue)."""
    h = np.asarray(h, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    K = h.shape[-1]
    assert r.shape[-1] == K + N - 1
    out = np.zeros(np.broadcast_shapes(h.shape[:-1], r.shape[:-1]) + (N,))
    for k in range(N):
        out[..., k] = np.sum(h * r[..., k:k + K], axis=-1)
    return out


def huber(z, delta: float):
    """L_delta(z) = z^2/2 if |z| <= delta else delta (|z| - delta/2)."""
    z = np.asarray(z, dtype=np.float64)
    a = np.abs(z)
    return np.where(a <= delta, 0.5 * z * z, delta * (a - 0.5 * delta))


def huber_grad(z, delta: float):
    """L_delta'(z) = z if |z| <= delta else delta sign(z)."""
    z = np.asarray(z, dtype=np.float64)
    return np.where(np.abs(z) <= delta, z, delta * np.sign(z))


def diff(h):
    """(D h)_j = h_{j+1} - h_j, j = 0 .. K-2."""
    h = np.asarray(h, dtype=np.float64)
    return h[..., 1:] - h[..., :-1]


def diff_adjoint(y):
    """D^T y for y of length K-1: (D^T y)_n = y_{n-1} [n >= 1] - y_n [n <= K-2]."""
    y = np.asarray(y, dtype=np.float64)
    K = y.shape[-1] + 1
    out = np.zeros(y.shape[:-1] + (K,))
    out[..., 1:] += y
    out[..., :-1] -= y
    return out


def bce_smooth(h, s, x, lam_tv: float, delta: float):
    """Smooth part of Eq. (6) and its gradients for C channels sharing one source.

    h [..., C, K], s [..., N], x [..., C, K+N-1]  ->  (F [...], grad_h [..., C, K], grad_s [..., N]).
    """
    h = np.asarray(h, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    K, N = h.shape[-1], s.shape[-1]
    r = conv_full(h, s[..., None, :]) - x                                   # r_i = h_i * s - x_i
    Dh = diff(h)
    F = np.sum(r * r, axis=(-2, -1)) + (lam_tv / delta) * np.sum(huber(Dh, delta), axis=(-2, -1))
    gh = 2.0 * conv_adjoint_h(s[..., None, :], r, K) + (lam_tv / delta) * diff_adjoint(huber_grad(Dh, delta))
    gs = 2.0 * np.sum(conv_adjoint_s(h, r, N), axis=-2)
    return F, gh, gs
