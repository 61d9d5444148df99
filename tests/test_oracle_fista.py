"""Oracle pins for FISTA around grad f (P:117, P:174 use 2500 FISTA iterations).

Pinned by what mathematics fixes, not by the oracle itself:
  * soft threshold: closed form on hand values;
  * power iteration: bounded by and converging to lambda_max of the dense (R W)^T (R W);
  * lasso optimality: lambda >= ||(R W)^T b||_inf  =>  the minimiser is 0 and FISTA returns 0;
  * convergence: after many iterations the KKT conditions of min 1/2||RWx-b||^2 + lambda||x||_1 hold,
    checked with the dense matrix (R W) assembled column by column;
  * momentum sequence t_k: the closed-form recursion t_{k+1} = (1 + sqrt(1 + 4 t_k^2)) / 2;
  * the W-dagger-closed gradient: equal to the true gradient for orthogonal filters
    under zero / periodic BC (W*_zpd = W-dagger_zpd for orthogonal wavelets), different
    for biorthogonal CDF 9/7 under symmetric BC, and equal to the dense A R^T (R W x - b) with A
    the assembled analysis matrix.
"""
import numpy as np
import pytest

H, W, J, FILT, BC = 12, 10, 2, "db2", "symmetric"


@pytest.fixture(scope="module")
def dense(oracle_lib):
    O = oracle_lib
    p = O.layout(H, W, J, FILT, BC).p
    Wm = O.synthesize(np.eye(p), H, W, J, FILT, BC).reshape(p, H * W)         # row i = W e_i
    RW = np.stack([O.blur(Wm[i].reshape(H, W)).ravel() for i in range(p)], 1)  # (hw, p)
    return O, p, RW


def test_soft_threshold_closed_form(oracle_lib):
    O = oracle_lib
    v = np.array([-3.0, -1.0, -0.5, 0.0, 0.25, 2.0])
    np.testing.assert_array_equal(O.soft_threshold(v, 1.0), [-2.0, 0.0, 0.0, 0.0, 0.0, 1.0])


def test_lipschitz_power_iteration(dense):
    O, p, RW = dense
    lmax = np.linalg.eigvalsh(RW.T @ RW).max()
    v0 = np.random.default_rng(0).standard_normal(p)
    e10 = O.lipschitz(v0, H, W, J, FILT, BC, 10)
    e300 = O.lipschitz(v0, H, W, J, FILT, BC, 300)
    assert e10 <= lmax * (1 + 1e-12) and e300 <= lmax * (1 + 1e-12)
    assert e300 >= e10 - 1e-12
    assert abs(e300 - lmax) <= 1e-9 * lmax


def test_fista_zero_solution_when_lambda_large(dense):
    O, p, RW = dense
    b = np.random.default_rng(1).standard_normal((1, H, W))
    lam = 1.01 * np.abs(RW.T @ b.ravel()).max()
    lip = np.linalg.eigvalsh(RW.T @ RW).max()
    x, _, _, trace = O.fista(np.zeros((1, p)), b, J, FILT, BC, lam, lip, 5)
    assert np.all(x == 0.0)
    np.testing.assert_allclose(trace, 0.5 * np.sum(b ** 2), rtol=1e-12)


def test_fista_kkt_at_convergence(dense):
    O, p, RW = dense
    rng = np.random.default_rng(2)
    xt = np.where(rng.random(p) < 0.2, rng.standard_normal(p), 0.0)
    b = (RW @ xt + 1e-3 * rng.standard_normal(H * W)).reshape(1, H, W)
    lam = 0.05 * np.abs(RW.T @ b.ravel()).max()
    lip = np.linalg.eigvalsh(RW.T @ RW).max()
    x, _, _, trace = O.fista(np.zeros((1, p)), b, J, FILT, BC, lam, lip, 3000)
    x = x.ravel()
    g = RW.T @ (RW @ x - b.ravel())                 # dense gradient, independent of the oracle's fast path
    nz = x != 0
    assert nz.any()
    np.testing.assert_allclose(g[nz] + lam * np.sign(x[nz]), 0.0, atol=1e-6 * lam + 1e-9)
    assert np.all(np.abs(g[~nz]) <= lam * (1 + 1e-6))
    assert trace[-1] <= trace[0]                    # FISTA is not monotone, but ends below its start


def test_momentum_sequence(oracle_lib):
    O = oracle_lib
    t = 1.0
    g = np.zeros(3)
    for k in range(1, 6):
        _, _, t_new = O.fista_update(g, g, g, t, 0.0, 1.0)
        assert t_new == pytest.approx((1 + np.sqrt(1 + 4 * t * t)) / 2)
        assert t_new > t and t_new >= (k + 1) / 2
        t = t_new


@pytest.mark.parametrize("filt", ["haar", "db2", "db4"])
@pytest.mark.parametrize("bc", ["zero", "periodic"])
def test_pinv_gradient_is_true_gradient_for_orthogonal(oracle_lib, filt, bc):
    O = oracle_lib
    h, w, j = 16, 24, 2
    p = O.layout(h, w, j, filt, bc).p
    rng = np.random.default_rng(3)
    x, b = rng.standard_normal((2, p)), rng.standard_normal((2, h, w))
    gt, ft = O.grad(x, b, j, filt, bc)
    gp, fp = O.grad(x, b, j, filt, bc, adjoint="pinv")
    np.testing.assert_allclose(gp, gt, rtol=0, atol=1e-12 * np.abs(gt).max())
    np.testing.assert_array_equal(fp, ft)


def test_pinv_gradient_dense_and_differs_for_biorthogonal(oracle_lib):
    O = oracle_lib
    h, w, j, filt, bc = 14, 12, 1, "cdf97", "symmetric"
    p = O.layout(h, w, j, filt, bc).p
    E = np.eye(h * w).reshape(h * w, h, w)
    A = O.analyze(E, j, filt, bc).T                                            # (p, hw): column k = W-dagger e_k
    Wm = O.synthesize(np.eye(p), h, w, j, filt, bc).reshape(p, h * w).T        # (hw, p)
    Rm = O.blur(E).reshape(h * w, h * w).T                                     # (hw, hw)
    rng = np.random.default_rng(4)
    x, b = rng.standard_normal(p), rng.standard_normal((h, w))
    r = Rm @ (Wm @ x) - b.ravel()
    gp, _ = O.grad(x[None], b[None], j, filt, bc, adjoint="pinv")
    np.testing.assert_allclose(gp[0], A @ (Rm.T @ r), atol=1e-11 * np.abs(gp).max())
    gt, _ = O.grad(x[None], b[None], j, filt, bc)
    assert np.linalg.norm(gp - gt) > 1e-3 * np.linalg.norm(gt)
