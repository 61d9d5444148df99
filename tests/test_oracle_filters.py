"""Oracle pins: filter banks (closed forms, published digits, textbook invariants)."""
from math import sqrt

import numpy as np
import pytest

from golden_io import load
from oracle.filters import cdf97_h, daubechies_h, filter_bank, gaussian_taps


def test_db2_closed_form():
    s3 = sqrt(3.0)
    ref = np.array([1 + s3, 3 + s3, 3 - s3, 1 - s3]) / (4 * sqrt(2.0))
    np.testing.assert_allclose(daubechies_h(2), ref, rtol=0, atol=1e-15)


def test_cdf97_published_digits():
    g = load("filters.txt")
    h9, h7 = cdf97_h()
    np.testing.assert_allclose(h9[4:] / sqrt(2.0), g["cdf97_analysis_lowpass_unitdc"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(h7[3:] * sqrt(2.0), g["cdf97_synthesis_lowpass_dc2"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(h9, h9[::-1], atol=1e-15)
    np.testing.assert_allclose(h7, h7[::-1], atol=1e-15)


@pytest.mark.parametrize("name,N", [("haar", 1), ("db2", 2), ("db4", 4), ("db8", 8)])
def test_daubechies_invariants(name, N):
    fb = filter_bank(name)
    assert fb.L == 2 * N
    lo, hi = fb.a_lo, fb.a_hi
    assert abs(lo.sum() - sqrt(2.0)) < 1e-14
    assert abs(hi.sum()) < 1e-14
    for k in range(N):                      # <lo, shift_2k lo> = delta_k ; <lo, shift_2k hi> = 0
        assert abs(np.dot(lo[2 * k:], lo[:fb.L - 2 * k]) - (1.0 if k == 0 else 0.0)) < 1e-14
        assert abs(np.dot(lo[2 * k:], hi[:fb.L - 2 * k])) < 1e-14
        assert abs(np.dot(hi[2 * k:], lo[:fb.L - 2 * k])) < 1e-14
    j = np.arange(fb.L, dtype=np.float64)
    for q in range(N + 1):                   # N vanishing moments exactly
        mom = np.sum(j ** q * hi)
        scale = np.sum(j ** q * np.abs(hi))
        if q < N:
            assert abs(mom) < 1e-12 * scale, (q, mom)
        else:
            assert abs(mom) > 1e-3 * scale
    # minimum phase: all zeros of h(z) other than z = -1 inside the unit circle
    h = daubechies_h(N)
    if N > 1:
        rts = np.roots(h)
        inner = rts[np.abs(rts + 1) > 0.2]      # the N-fold zero at -1 is ill-conditioned
        assert inner.size == N - 1
        assert np.all(np.abs(inner) < 1)
    np.testing.assert_array_equal(fb.d_lo, fb.a_lo)
    np.testing.assert_array_equal(fb.d_hi, fb.a_hi)


def test_cdf97_bank():
    fb = filter_bank("cdf97")
    assert fb.L == 10 and not fb.orthogonal
    assert np.count_nonzero(fb.a_lo) == 9 and np.count_nonzero(fb.d_lo) == 7
    assert np.count_nonzero(fb.a_hi) == 7 and np.count_nonzero(fb.d_hi) == 9
    j = np.arange(10.0)
    for hi in (fb.a_hi, fb.d_hi):
        for q in range(4):
            assert abs(np.sum(j ** q * hi)) < 1e-12 * np.sum(j ** q * np.abs(hi))
        assert abs(np.sum(j ** 4 * hi)) > 1e-3 * np.sum(j ** 4 * np.abs(hi))
    # biorthogonality of the two lowpasses on even shifts (same centre, index 5)
    for k in range(-4, 5):
        lhs = sum(fb.a_lo[n] * fb.d_lo[n + 2 * k] for n in range(10) if 0 <= n + 2 * k < 10)
        assert abs(lhs - (1.0 if k == 0 else 0.0)) < 1e-14


def test_gaussian_taps():
    k = gaussian_taps(15, 3.0)
    assert k.size == 15 and abs(k.sum() - 1.0) < 1e-15
    np.testing.assert_array_equal(k, k[::-1])
    # ratio of neighbouring samples of exp(-t^2/18): k[t+1]/k[t] = exp(-(2t+1)/18)
    t = np.arange(-7, 7)
    np.testing.assert_allclose(k[1:] / k[:-1], np.exp(-(2 * t + 1) / 18.0), rtol=1e-14)
    assert gaussian_taps(1, 1.0).tolist() == [1.0]
