"""Oracle filter banks (fp64, numpy).  TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / reference
leg may import anything under `oracle/`.  The product path (the CUDA library under
`paper_1707_02018_b200/`) computes its own filter banks with an independent
algorithm (C++ Durand-Kerner root finding + Cardano); nothing here is shared.

The paper never lists its filter coefficients; it names the families it uses:
  * "orthogonal wavelets (e.g., Haar and more generally Daubechies wavelets)"
    PAPER.md §"The adjoint for orthogonal wavelets",
  * "a three-stage CDF 9/7 discrete wavelet transform",
and BASELINE.json configs (BJ:7-11) name db2, db4, db8 and CDF 9/7
("standard closed-form coefficients").  The constructions below are the textbook
ones (Daubechies 1988 spectral factorisation; Cohen-Daubechies-Feauveau 9/7 from the
roots of P_4), restated from SURVEY.md §8(c) C.1 "Filters".

Array conventions (reading R4/R5):
  * every bank lives in a common frame of L taps (L even);
  * analysis is a convolution with the odd phase kept:
        A_f(yhat)[k] = sum_{j<L} f[j] * yhat[2k+1-j]
  * a_lo, a_hi = analysis pair (W-dagger); d_lo, d_hi = dual / synthesis pair
    (W and W* use these, paper Eq. (4): W* = W~dagger_zpd (E^dagger)*);
  * unified highpass rule: a_hi[j] = (-1)^(j+1) d_lo[L-1-j],
                           d_hi[j] = (-1)^(j+1) a_lo[L-1-j].
Parity unpinned: none -- every bank is pinned in tests/test_oracle_filters.py
(db2 closed form, CDF 9/7 published digits, orthonormality, biorthogonality,
vanishing moments).
"""
from __future__ import annotations

from dataclasses import dataclass
from math import comb, sqrt

import numpy as np

__all__ = ["FilterBank", "filter_bank", "daubechies_h", "cdf97_h", "FILTERS", "gaussian_taps"]


@dataclass(frozen=True)
class FilterBank:
    name: str
    L: int               # common frame length (even)
    a_lo: np.ndarray     # analysis lowpass   (W-dagger)
    a_hi: np.ndarray     # analysis highpass  (W-dagger)
    d_lo: np.ndarray     # dual lowpass       (W, W*)
    d_hi: np.ndarray     # dual highpass      (W, W*)
    orthogonal: bool


def _poly_from_roots_zinv(roots):
    """Coefficients (in powers of z^-1, c[0] = z^0) of prod (1 - r z^-1)."""
    c = np.array([1.0 + 0j])
    for r in roots:
        c = np.convolve(c, np.array([1.0, -r]))
    return c


def daubechies_h(N: int) -> np.ndarray:
    """Minimum-phase Daubechies lowpass h (length 2N, sum sqrt(2)).

    P_N(y) = sum_{k<N} C(N-1+k, k) y^k with y = sin^2(w/2) = (2 - z - 1/z)/4.
    Each root y_r of P_N maps to the roots of z^2 - (2 - 4 y_r) z + 1; the one
    inside the unit circle is kept (minimum phase).  h(z) ∝ (1+z^-1)^N prod(1 - z_r z^-1).
    """
    if N == 1:
        return np.array([1.0, 1.0]) / sqrt(2.0)
    pcoef = [comb(N - 1 + k, k) for k in range(N)]          # ascending powers of y
    yroots = np.roots(pcoef[::-1])                           # companion-matrix eigenvalues
    zroots = []
    for yr in yroots:
        b = 2.0 - 4.0 * yr
        disc = np.sqrt(b * b - 4.0 + 0j)
        z1, z2 = (b + disc) / 2.0, (b - disc) / 2.0
        zroots.append(z1 if abs(z1) < 1.0 else z2)
    c = _poly_from_roots_zinv([-1.0] * N + zroots)
    h = np.real(c)
    return h * (sqrt(2.0) / h.sum())


def _cos4_times(ypoly_roots):
    """Symmetric filter ∝ cos^4(w/2) * prod (y - y_r), y = (2 - z - 1/z)/4.

    Returned as real coefficients of z^-k, centred (zero phase), sum sqrt(2).
    """
    # cos^2(w/2) = (2 + z + 1/z)/4 -> coefficients over z^{-1..1}: [1, 2, 1]/4
    c2 = np.array([1.0, 2.0, 1.0]) / 4.0
    f = np.convolve(c2, c2)                                   # cos^4
    for yr in ypoly_roots:
        # y - y_r = (-z + 2 - 1/z)/4 - y_r  -> [-1/4, 1/2 - y_r, -1/4]
        f = np.convolve(f, np.array([-0.25, 0.5 - yr, -0.25]))
    f = np.real(f)
    return f * (sqrt(2.0) / f.sum())


def cdf97_h():
    """CDF 9/7 lowpass pair (h9 = analysis, 7 taps = synthesis), sum sqrt(2) each.

    Roots of P_4(y) = 1 + 4y + 10y^2 + 20y^3: the real root goes to the 7-tap
    filter, the complex pair to the 9-tap filter.
    """
    yroots = np.roots([20.0, 10.0, 4.0, 1.0])
    real = [r for r in yroots if abs(r.imag) < 1e-12]
    cplx = [r for r in yroots if abs(r.imag) >= 1e-12]
    assert len(real) == 1 and len(cplx) == 2
    h7 = _cos4_times([real[0].real])
    h9 = _cos4_times(cplx)
    assert h7.size == 7 and h9.size == 9
    return h9, h7


def _highpass(L, lo_other):
    j = np.arange(L)
    return ((-1.0) ** (j + 1)) * lo_other[L - 1 - j]


def filter_bank(name: str) -> FilterBank:
    name = name.lower()
    if name in ("haar", "db1", "db2", "db4", "db8"):
        N = 1 if name in ("haar", "db1") else int(name[2:])
        h = daubechies_h(N)
        L = 2 * N
        lo = h[::-1].copy()                                   # a_lo = d_lo = reverse(h)
        hi = _highpass(L, lo)
        return FilterBank(name, L, lo, hi, lo.copy(), hi.copy(), True)
    if name in ("cdf97", "cdf9/7", "bior4.4"):
        h9, h7 = cdf97_h()
        L = 10                                                # common 10-tap frame (reading R3)
        a_lo = np.zeros(L); a_lo[1:10] = h9
        d_lo = np.zeros(L); d_lo[2:9] = h7
        a_hi = _highpass(L, d_lo)
        d_hi = _highpass(L, a_lo)
        return FilterBank("cdf97", L, a_lo, a_hi, d_lo, d_hi, False)
    raise ValueError(f"unknown filter bank {name!r}")


FILTERS = ("haar", "db2", "db4", "db8", "cdf97")


def gaussian_taps(ntaps: int = 15, sigma: float = 3.0) -> np.ndarray:
    """Blur PSF per axis (reading R12): k[t] = exp(-t^2 / (2 sigma^2)) / sum, t = -h..h.

    PAPER.md P:31 ("a Gaussian point spread function (PSF) under symmetric
    (reflexive) boundary conditions"); size/sigma from BASELINE.json config 5.
    """
    if ntaps % 2 != 1 or ntaps < 1:
        raise ValueError("ntaps must be odd")
    h = ntaps // 2
    t = np.arange(-h, h + 1, dtype=np.float64)
    k = np.exp(-(t * t) / (2.0 * sigma * sigma))
    return k / k.sum()
