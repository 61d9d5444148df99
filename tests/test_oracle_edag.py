"""Oracle pins for the paper-literal symmetric variant (bc = "symmetric_edag", reading R1 "P").

PAPER.md §"The adjoint for symmetric extension" and Eq. (4) define
W*_P = W~dagger_zpd (E_sym^dagger)*; §"Example 1" says the pseudoinverse trick's
"error is introduced through E ~ (E^dagger)*".  The oracle evaluates (E_sym^dagger)* through a
per-level multiplicity table (oracle.c `cinv_table`).  These pins rebuild every level from
matrices that share nothing with that table:

  * E_sym is written out from the displayed matrix of P:82 (half-point reflection) and checked
    against the oracle's `extend` (itself pinned to the printed N = 5 example);
  * (E_sym^dagger)* is numpy.linalg.pinv(E_sym)^T -- brute force, no multiplicity counting;
  * the analysis core A_f[k, t] = f[2k+1-t] (reading R5) is assembled as a dense matrix.

A wrong multiplicity window (L instead of L-1), weights applied on one axis only, a level
whose weights come from the wrong length, or the 1/3 regime (n < 2L'; reading R10)
handled as 1/2 each fail one of these tests.
"""
import numpy as np
import pytest

from oracle.filters import filter_bank


def E_sym(n, Lp):
    """Half-point symmetric extension onto t in [-Lp, n+Lp), the matrix displayed at P:82."""
    E = np.zeros((n + 2 * Lp, n))
    for t in range(-Lp, n + Lp):
        s = t
        while s < 0 or s >= n:          # reflect until inside (only one reflection when n >= Lp)
            s = -1 - s if s < 0 else 2 * n - 1 - s
        E[t + Lp, s] = 1.0
    return E


def A_core(f, n, Lp):
    """Analysis core over the extended vector: out[k] = sum_j f[j] yhat[2k+1-j], k < m (R5)."""
    L = len(f)
    m = (n + L - 1) // 2
    A = np.zeros((m, n + 2 * Lp))
    for k in range(m):
        for j in range(L):
            t = 2 * k + 1 - j
            A[k, t + Lp] += f[j]
    return A


def level_mats(fb, n, ext):
    """(lo, hi) per-axis matrices of one level: A_f X with X = (E^dagger)* (pinv) or E (sym)."""
    Lp = fb.L - 1
    E = E_sym(n, Lp)
    X = np.linalg.pinv(E).T if ext == "pinv" else E
    lo = fb.d_lo if ext == "pinv" else fb.a_lo
    hi = fb.d_hi if ext == "pinv" else fb.a_hi
    return A_core(lo, n, Lp) @ X, A_core(hi, n, Lp) @ X


def multilevel_numpy(Y, J, fb, ext):
    """Packed LL_J, (LH_j, HL_j, HH_j)_{j=J..1} (reading R7) built from the per-axis matrices;
    subband XY = axis-0 filter X, axis-1 filter Y (reading R8)."""
    details = []
    LL = Y
    for _ in range(J):
        n0, n1 = LL.shape
        M0lo, M0hi = level_mats(fb, n0, ext)
        M1lo, M1hi = level_mats(fb, n1, ext)
        details.append((M0lo @ LL @ M1hi.T, M0hi @ LL @ M1lo.T, M0hi @ LL @ M1hi.T))
        LL = M0lo @ LL @ M1lo.T
    parts = [LL.ravel()]
    for lh, hl, hh in reversed(details):
        parts += [lh.ravel(), hl.ravel(), hh.ravel()]
    return np.concatenate(parts)


SHAPES = [  # (h, w, J): interior, odd sizes, and the n < 2L' (1/3) regime at a level input
    (13, 11, 1), (13, 11, 2), (9, 12, 2), (5, 7, 1), (17, 19, 2),
]


def _ok(O, h, w, J, filt):
    try:
        O.layout(h, w, J, filt, "symmetric_edag")
        return True
    except ValueError:
        return False


def test_E_sym_matches_oracle_extend(oracle_lib):
    O = oracle_lib
    for n, Lp in [(5, 2), (7, 3), (4, 3), (16, 7)]:
        E = np.stack([O.extend(np.eye(n)[i], Lp, "symmetric") for i in range(n)], axis=1)
        np.testing.assert_array_equal(E, E_sym(n, Lp))


@pytest.mark.parametrize("filt", ("haar", "db2", "db4", "cdf97"))
@pytest.mark.parametrize("h,w,J", SHAPES)
def test_edag_adjoint_equals_pinv_construction(oracle_lib, filt, h, w, J):
    """W*_P y from the oracle == the level-by-level product with numpy's pinv(E_sym)^T."""
    O = oracle_lib
    if not _ok(O, h, w, J, filt):
        pytest.skip("chain not formable")
    fb = filter_bank(filt)
    rng = np.random.default_rng(100 + h * w + J)
    Y = rng.standard_normal((h, w))
    got = O.adjoint(Y, J, filt, "symmetric_edag")
    want = multilevel_numpy(Y, J, fb, "pinv")
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-13 * max(1.0, np.abs(want).max()))


@pytest.mark.parametrize("filt", ("haar", "db2", "db4", "cdf97"))
@pytest.mark.parametrize("h,w,J", SHAPES)
def test_edag_synthesis_is_transpose_of_pinv_construction(oracle_lib, filt, h, w, J):
    """W_P x == (dense W*_P)^T x, the dense matrix assembled from the numpy construction."""
    O = oracle_lib
    if not _ok(O, h, w, J, filt):
        pytest.skip("chain not formable")
    fb = filter_bank(filt)
    cols = [multilevel_numpy(np.eye(h * w)[i].reshape(h, w), J, fb, "pinv") for i in range(h * w)]
    Wstar = np.stack(cols, axis=1)                                   # (p, hw)
    rng = np.random.default_rng(7 + h + w)
    x = rng.standard_normal(Wstar.shape[0])
    got = O.synthesize(x, h, w, J, filt, "symmetric_edag").ravel()
    np.testing.assert_allclose(got, Wstar.T @ x, rtol=0, atol=1e-13 * max(1.0, np.abs(x).max()))


@pytest.mark.parametrize("filt", ("haar", "db2", "db4", "db8"))
@pytest.mark.parametrize("n1", [24, 11, 5, 4])
def test_p106_error_through_extension(oracle_lib, filt, n1):
    """P:106 for orthogonal banks (a = d): W*_P - W-dagger = A_a ((E^dagger)* - E).

    With an image Y = u v^T whose column factor u vanishes within L' of the top/bottom edges,
    (E^dagger)* u = E u along axis 0, so every subband of the difference is the outer product
    of (A_X E u) with the 1-D error A_Y ((E^dagger)* - E) v along axis 1.  n1 = 5, 4 < 2L'
    for db2 reach the 1/3 regime."""
    O = oracle_lib
    fb = filter_bank(filt)
    assert fb.orthogonal
    Lp = fb.L - 1
    if n1 < Lp:
        pytest.skip("E_sym needs n >= L'")
    n0 = 2 * Lp + 8
    rng = np.random.default_rng(n1 + fb.L)
    u = np.zeros(n0)
    u[Lp:n0 - Lp] = rng.standard_normal(n0 - 2 * Lp)
    v = rng.standard_normal(n1)
    Y = np.outer(u, v)
    diff = O.adjoint(Y, 1, filt, "symmetric_edag") - O.analyze(Y, 1, filt, "symmetric")
    E0, E1 = E_sym(n0, Lp), E_sym(n1, Lp)
    P1 = np.linalg.pinv(E1).T
    np.testing.assert_allclose(np.linalg.pinv(E0).T @ u, E0 @ u, atol=1e-14)   # premise on axis 0
    a0 = {X: A_core(f, n0, Lp) @ E0 @ u for X, f in (("L", fb.a_lo), ("H", fb.a_hi))}
    e1 = {X: A_core(f, n1, Lp) @ (P1 - E1) @ v for X, f in (("L", fb.a_lo), ("H", fb.a_hi))}
    m0, m1 = len(a0["L"]), len(e1["L"])
    want = np.concatenate([np.outer(a0[X], e1[Yb]).ravel() for X, Yb in (("L", "L"), ("L", "H"), ("H", "L"), ("H", "H"))])
    assert diff.size == 4 * m0 * m1
    np.testing.assert_allclose(diff, want, rtol=0, atol=1e-13 * max(1.0, np.abs(want).max()))
    # the error is real: it does not vanish for a generic v (the trick is an approximation)
    assert np.abs(want).max() > 1e-3
