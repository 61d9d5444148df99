"""Oracle pins: the multi-level operators W, W*, W-dagger, R, R* and grad f.

Every check here is fixed by the paper or by mathematics, not by the oracle itself:
  * dense transpose: W assembled column by column equals the transpose of W* assembled
    column by column (W* is computed by the analysis loops, W by the scatter loops);
  * adjoint identity <W x, y> = <x, W* y>;
  * perfect reconstruction W W-dagger b = b (BASELINE.json north_star);
  * orthogonal + periodic: W* = W-dagger = W^{-1} (BJ north_star), Parseval;
  * orthogonal + zero: W*_zpd = W-dagger_zpd, isometry;
  * CDF 9/7 + symmetric: W* != W-dagger (BJ config 3);
  * constant image under symmetric / periodic BC has zero details (vanishing moment 0);
  * coefficient-length chains quoted by BASELINE.json configs 1-5;
  * R: R 1 = 1, R = R^T, R* (fold form) = R, R = (C^T diag(lambda) C) per axis with the
    orthonormal DCT-II from scipy (Hansen/Nagy/O'Leary reflexive-BC diagonalisation), delta PSF = I;
  * grad f: dense W^T R^T (R W x - b), central finite differences, zero at b = R W x.
"""
import numpy as np
import pytest
import scipy.fft

from oracle.filters import FILTERS, filter_bank, gaussian_taps

BCS = ("zero", "periodic", "symmetric", "symmetric_edag")


def _shape(bc, filt):
    L = filter_bank(filt).L
    if bc == "periodic":
        return 16, 24, 2
    if bc.startswith("symmetric") and L == 16:
        return 17, 19, 2
    return 13, 11, 2


def dense_W(O, h, w, J, filt, bc):
    p = O.layout(h, w, J, filt, bc).p
    return O.synthesize(np.eye(p), h, w, J, filt, bc).reshape(p, h * w).T       # (hw, p)


def dense_Wstar(O, h, w, J, filt, bc):
    imgs = np.eye(h * w).reshape(h * w, h, w)
    return O.adjoint(imgs, J, filt, bc).T                                       # (p, hw)


def dense_Wdag(O, h, w, J, filt, bc):
    imgs = np.eye(h * w).reshape(h * w, h, w)
    return O.analyze(imgs, J, filt, bc).T


@pytest.mark.parametrize("filt", FILTERS)
@pytest.mark.parametrize("bc", BCS)
def test_dense_transpose_and_adjoint_identity(oracle_lib, filt, bc):
    O = oracle_lib
    h, w, J = _shape(bc, filt)
    Wm = dense_W(O, h, w, J, filt, bc)
    Ws = dense_Wstar(O, h, w, J, filt, bc)
    assert np.abs(Wm.T - Ws).max() <= 1e-15 * max(1.0, np.abs(Wm).max()) * 4
    rng = np.random.default_rng(5)
    x = rng.standard_normal(Wm.shape[1])
    y = rng.standard_normal((h, w))
    Wx = O.synthesize(x, h, w, J, filt, bc)
    d = abs(np.vdot(Wx, y) - np.vdot(x, O.adjoint(y, J, filt, bc))) / (np.linalg.norm(Wx) * np.linalg.norm(y))
    assert d <= 1e-14


@pytest.mark.parametrize("filt", FILTERS)
@pytest.mark.parametrize("bc", ("zero", "periodic", "symmetric"))
@pytest.mark.parametrize("shape", [(32, 32, 3), (29, 35, 2), (40, 18, 1)])
def test_perfect_reconstruction(oracle_lib, filt, bc, shape):
    O = oracle_lib
    h, w, J = shape
    if bc == "periodic" and (h % (1 << J) or w % (1 << J)):
        pytest.skip("periodisation needs even lengths at every level")
    L = filter_bank(filt).L
    try:
        O.layout(h, w, J, filt, bc)
    except ValueError:
        pytest.skip("chain not formable")
    rng = np.random.default_rng(1)
    b = rng.standard_normal((2, h, w))
    rec = O.synthesize(O.analyze(b, J, filt, bc), h, w, J, filt, bc)
    assert np.abs(rec - b).max() <= 1e-13 * (1 + L)


@pytest.mark.parametrize("filt", ("haar", "db2", "db4", "db8"))
def test_orthogonal_periodic_is_inverse(oracle_lib, filt):
    O = oracle_lib
    h, w, J = 32, 48, 2
    rng = np.random.default_rng(2)
    y = rng.standard_normal((h, w))
    a = O.analyze(y, J, filt, "periodic")
    s = O.adjoint(y, J, filt, "periodic")
    np.testing.assert_allclose(s, a, rtol=0, atol=1e-13)
    assert abs(np.linalg.norm(a) - np.linalg.norm(y)) < 1e-12 * np.linalg.norm(y)      # Parseval
    x = rng.standard_normal(a.size)
    np.testing.assert_allclose(O.analyze(O.synthesize(x, h, w, J, filt, "periodic"), J, filt, "periodic"),
                               x, rtol=0, atol=1e-13)                                    # W^{-1} both sides


def test_cfg1_dense_4096(oracle_lib):
    """BASELINE.json config 1: 64x64 db2, 3 levels, periodic; W* vs the dense 4096x4096 W^T;
    orthogonal + periodic => W* = W-dagger = W^{-1}."""
    O = oracle_lib
    Wm = dense_W(O, 64, 64, 3, "db2", "periodic")
    assert Wm.shape == (4096, 4096)
    Ws = dense_Wstar(O, 64, 64, 3, "db2", "periodic")
    assert np.abs(Wm.T - Ws).max() < 1e-15
    np.testing.assert_allclose(Ws @ Wm, np.eye(4096), rtol=0, atol=1e-13)


@pytest.mark.parametrize("filt", ("haar", "db2", "db4", "db8"))
def test_orthogonal_zero_bc(oracle_lib, filt):
    """for orthogonal wavelets W*_zpd = W-dagger_zpd; W-dagger_zpd is an isometry."""
    O = oracle_lib
    rng = np.random.default_rng(3)
    y = rng.standard_normal((37, 30))
    a = O.analyze(y, 2, filt, "zero")
    np.testing.assert_allclose(O.adjoint(y, 2, filt, "zero"), a, rtol=0, atol=1e-13)
    assert abs(np.linalg.norm(a) - np.linalg.norm(y)) < 1e-12 * np.linalg.norm(y)
    # reading R1: the symmetric W* equals the zero-BC analysis for orthogonal banks
    np.testing.assert_allclose(O.adjoint(y, 2, filt, "symmetric"), a, rtol=0, atol=1e-13)


def test_cdf97_symmetric_adjoint_differs_from_analysis(oracle_lib):
    O = oracle_lib
    h, w, J = 24, 24, 2
    gap = np.abs(dense_Wstar(O, h, w, J, "cdf97", "symmetric") - dense_Wdag(O, h, w, J, "cdf97", "symmetric")).max()
    assert gap > 0.1


@pytest.mark.parametrize("filt", FILTERS)
@pytest.mark.parametrize("bc", ("symmetric", "periodic"))
def test_constant_image_zero_details(oracle_lib, filt, bc):
    O = oracle_lib
    h, w, J = (32, 32, 3) if bc == "periodic" else (35, 30, 2)
    lay = O.layout(h, w, J, filt, bc)
    x = O.analyze(np.full((h, w), 3.0), J, filt, bc)
    n_ll = lay.c0[J] * lay.c1[J]
    assert np.abs(x[n_ll:]).max() < 1e-12
    np.testing.assert_allclose(x[:n_ll], 3.0 * 2.0 ** J, rtol=1e-13)   # DC gain sqrt(2) per axis per level


@pytest.mark.parametrize("filt", ("db2", "db4", "cdf97"))
def test_edag_pr_only_in_interior(oracle_lib, filt):
    """Reading R1 / SURVEY §8(c) item 1: the paper-literal W_P = E_sym^dagger W_zpd reconstructs
    exactly away from the edges and not near them (documented behaviour, not a defect)."""
    O = oracle_lib
    L = filter_bank(filt).L
    h, w = 48, 40
    rng = np.random.default_rng(4)
    b = rng.standard_normal((h, w))
    err = np.abs(O.synthesize(O.analyze(b, 1, filt, "symmetric_edag"), h, w, 1, filt, "symmetric_edag") - b)
    m = L
    assert err[m:-m, m:-m].max() < 1e-13
    assert err.max() > 1e-3


def test_level_chains_of_baseline_configs(oracle_lib):
    O = oracle_lib
    # chains from BASELINE.json configs (floor((n+L-1)/2) zero/sym; n/2 periodic), SURVEY §8(a) table
    assert O.chain(64, 4, "periodic", 3) == [64, 32, 16, 8]
    assert O.chain(512, 8, "symmetric", 4) == [512, 259, 133, 70, 38]
    assert O.chain(2048, 10, "symmetric", 5) == [2048, 1028, 518, 263, 136, 72]
    assert O.chain(4096, 16, "zero", 6) == [4096, 2055, 1035, 525, 270, 142, 78]
    assert O.chain(4096, 10, "symmetric", 5) == [4096, 2052, 1030, 519, 264, 136]
    assert O.layout(64, 64, 3, "db2", "periodic").p == 4096
    assert O.layout(512, 512, 4, "db4", "symmetric").p == 274786
    assert O.layout(2048, 2048, 5, "cdf97", "symmetric").p == 4259055
    assert O.layout(4096, 4096, 6, "db8", "zero").p == 17013153
    assert O.layout(4096, 4096, 5, "cdf97", "symmetric").p == 16905967
    with pytest.raises(ValueError):
        O.chain(20, 4, "periodic", 3)          # odd length at level 3
    with pytest.raises(ValueError):
        O.chain(10, 16, "symmetric", 1)        # E_sym needs n >= L' = 15
    assert O.chain(15, 16, "symmetric", 3) == [15, 15, 15, 15]   # fixed point of floor((n+15)/2)


# ------------------------------------------------------------------------- blur
def _dense_blur(O, h, w, taps, adjoint=False):
    imgs = np.eye(h * w).reshape(h * w, h, w)
    f = O.blur_adjoint if adjoint else O.blur
    return f(imgs, taps).reshape(h * w, h * w).T


def test_blur_properties(oracle_lib):
    O = oracle_lib
    h, w = 24, 17
    k = gaussian_taps(15, 3.0)
    R = _dense_blur(O, h, w, k)
    Rs = _dense_blur(O, h, w, k, adjoint=True)
    np.testing.assert_allclose(R @ np.ones(h * w), 1.0, rtol=0, atol=1e-15)
    np.testing.assert_allclose(Rs, R.T, rtol=0, atol=1e-16)          # fold form is the transpose
    np.testing.assert_allclose(R, R.T, rtol=0, atol=1e-16)           # symmetric PSF: R* = R
    # DCT-II diagonalisation (reflexive BC, symmetric PSF): R_a = C^T diag(lam) C per axis,
    # lam_q = sum_t k[t] cos(pi q t / n)
    def axis(n):
        C = scipy.fft.dct(np.eye(n), type=2, norm="ortho", axis=0)
        t = np.arange(-7, 8)
        lam = np.array([np.sum(k * np.cos(np.pi * q * t / n)) for q in range(n)])
        return C.T @ np.diag(lam) @ C
    np.testing.assert_allclose(R, np.kron(axis(h), axis(w)), rtol=0, atol=1e-15)
    delta = np.zeros(15); delta[7] = 1.0
    img = np.random.default_rng(0).standard_normal((h, w))
    np.testing.assert_array_equal(O.blur(img, delta), img)


# ------------------------------------------------------------------------- grad
@pytest.mark.parametrize("filt,bc", [("haar", "symmetric"), ("cdf97", "symmetric"), ("db2", "periodic"),
                                     ("db4", "zero"), ("cdf97", "symmetric_edag")])
def test_grad(oracle_lib, filt, bc):
    O = oracle_lib
    h, w, J = (16, 16, 2) if bc == "periodic" else (15, 13, 2)
    rng = np.random.default_rng(6)
    Wm = dense_W(O, h, w, J, filt, bc)
    R = _dense_blur(O, h, w, gaussian_taps())
    x = rng.standard_normal(Wm.shape[1])
    b = rng.standard_normal((h, w))
    g, f = O.grad(x, b, J, filt, bc)
    r = R @ (Wm @ x) - b.ravel()
    np.testing.assert_allclose(g, Wm.T @ (R.T @ r), rtol=0, atol=1e-13)
    assert abs(f - 0.5 * r @ r) < 1e-12 * (r @ r)
    # central finite differences along a random direction
    e = rng.standard_normal(x.size)
    eps = 1e-5
    fp = O.grad(x + eps * e, b, J, filt, bc)[1]
    fm = O.grad(x - eps * e, b, J, filt, bc)[1]
    assert abs((fp - fm) / (2 * eps) - g @ e) < 1e-7 * (abs(g @ e) + 1)
    # exact data => zero gradient
    b0 = (R @ (Wm @ x)).reshape(h, w)
    g0, f0 = O.grad(x, b0, J, filt, bc)
    assert np.abs(g0).max() < 1e-13 and f0 < 1e-26


# ------------------------------------------------ (W-dagger)*: SURVEY §8(f) NEXT #2
@pytest.mark.parametrize("filt", FILTERS)
@pytest.mark.parametrize("bc", BCS)
def test_analyze_adjoint_is_dense_transpose(oracle_lib, filt, bc):
    """(W-dagger)* (scatter loops with the analysis filters + E_bc^T fold) equals the transpose of
    W-dagger assembled column by column from the analysis loops; adjoint identity."""
    O = oracle_lib
    h, w, J = _shape(bc, filt)
    A = dense_Wdag(O, h, w, J, filt, bc)                                         # (p, hw)
    p = A.shape[0]
    At = O.analyze_adjoint(np.eye(p), h, w, J, filt, bc).reshape(p, h * w).T     # (hw, p)
    assert np.abs(A.T - At).max() <= 1e-15 * max(1.0, np.abs(A).max()) * 8
    rng = np.random.default_rng(17)
    x = rng.standard_normal(p)
    y = rng.standard_normal((h, w))
    lhs = np.vdot(O.analyze(y, J, filt, bc), x)
    rhs = np.vdot(y, O.analyze_adjoint(x, h, w, J, filt, bc))
    assert abs(lhs - rhs) <= 1e-13 * np.linalg.norm(x) * np.linalg.norm(y)


@pytest.mark.parametrize("filt", [f for f in FILTERS if filter_bank(f).orthogonal])
def test_analyze_adjoint_orthogonal_periodic_is_W(oracle_lib, filt):
    """Orthogonal + periodic: W-dagger = W* = W^{-1} (BJ north_star), so (W-dagger)* = W."""
    O = oracle_lib
    h, w, J = 16, 24, 2
    x = np.random.default_rng(3).standard_normal(O.layout(h, w, J, filt, "periodic").p)
    np.testing.assert_allclose(O.analyze_adjoint(x, h, w, J, filt, "periodic"),
                               O.synthesize(x, h, w, J, filt, "periodic"), rtol=0, atol=1e-13)


def test_analyze_adjoint_symmetric_differs_from_W(oracle_lib):
    """Under symmetric BC, (W-dagger)* folds reflect-add with the analysis filters, so for CDF 9/7
    it differs from W (crop, dual filters) by far more than rounding: a guard against swapping them."""
    O = oracle_lib
    h, w, J = 24, 20, 2
    x = np.random.default_rng(4).standard_normal(O.layout(h, w, J, "cdf97", "symmetric").p)
    a = O.analyze_adjoint(x, h, w, J, "cdf97", "symmetric")
    b = O.synthesize(x, h, w, J, "cdf97", "symmetric")
    assert np.linalg.norm(a - b) > 0.05 * np.linalg.norm(b)
