"""GPU FISTA against the fp64 oracle on identical inputs.

Tolerances (DESIGN.md §3 "FISTA"): the fused update is elementwise, so it matches the oracle's
update to rounding (fp64 1e-13, fp32 2e-6, like the operators).  K iterations compose K gradients
and K soft-thresholds; fp64 stays at 1e-11 after 10 iterations; fp32 at 1e-4 (per-iteration
operator error ~1e-7 relative, grown by the iteration and by coefficients crossing the threshold
in one precision and not the other).  The power iteration converges to lambda_max of the dense
(R W)^T (R W) from below.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1707_02018_b200 import inputs, wl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def dev(torch, a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=getattr(torch, dtype))


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-13), ("float32", 2e-6)])
def test_fista_update_matches_oracle(torch, dtype, tol):
    plan = wl.Plan(37, 45, 2, "cdf97", "symmetric", dtype)
    rng = np.random.default_rng(0)
    B = 2
    g, x, y = (inputs.cast(rng.standard_normal((B, plan.p_valid)), dtype) for _ in range(3))
    t, lam, lip = 1.7, 0.3, 2.5
    xo, yo, to = O.fista_update(g, x, y, t, lam, lip)
    gd, xd, yd = (dev(torch, plan.from_packed(a), dtype) for a in (g, x, y))
    t_new = wl.fista_update(plan, gd, xd, yd, t, lam, lip)
    assert t_new == pytest.approx(to, rel=1e-15)
    assert rel(plan.to_packed(xd.double().cpu().numpy()), xo) <= tol
    assert rel(plan.to_packed(yd.double().cpu().numpy()), yo) <= tol
    pad = np.setdiff1d(np.arange(plan.p_alloc), plan.to_packed(np.arange(plan.p_alloc)[None])[0].astype(np.int64))
    assert np.all(xd.cpu().numpy()[:, pad] == 0) and np.all(yd.cpu().numpy()[:, pad] == 0)


@pytest.mark.parametrize("filt,bc", [("cdf97", "symmetric"), ("haar", "symmetric"), ("db4", "zero")])
@pytest.mark.parametrize("dtype,tol", [("float64", 1e-11), ("float32", 1e-4)])
def test_fista_iterations_match_oracle(torch, filt, bc, dtype, tol):
    h, w, J, B, K = 40, 36, 3, 2, 10
    plan = wl.Plan(h, w, J, filt, bc, dtype)
    blur = wl.Blur(h, w, 15, 3.0, dtype=dtype)
    rng = np.random.default_rng(5)
    b = inputs.cast(O.blur(inputs.blobs(rng, B, h, w, 8)) + 1e-3 * rng.standard_normal((B, h, w)), dtype)
    lam, lip = 2e-3, 1.05
    x, y, t, _ = O.fista(np.zeros((B, plan.p_valid)), b, J, filt, bc, lam, lip, K)
    xg, yg, tg = wl.fista(plan, blur, dev(torch, b, dtype), lam, K, lip=lip)
    assert tg == pytest.approx(t, rel=1e-14)
    assert rel(plan.to_packed(xg.double().cpu().numpy()), x) <= tol
    assert rel(plan.to_packed(yg.double().cpu().numpy()), y) <= tol


def test_fista_zero_solution_when_lambda_large(torch):
    h, w, J = 32, 32, 2
    plan = wl.Plan(h, w, J, "db2", "symmetric", "float64")
    blur = wl.Blur(h, w, 15, 3.0, dtype="float64")
    b = np.random.default_rng(1).standard_normal((1, h, w))
    lam = 1.01 * np.abs(O.grad(np.zeros((1, plan.p_valid)), b, J, "db2", "symmetric")[0]).max()
    xg, _, _ = wl.fista(plan, blur, dev(torch, b, "float64"), lam, 5, lip=1.0)
    assert float(xg.abs().max()) == 0.0


def test_lipschitz_matches_dense_eigenvalue(torch):
    h, w, J, filt, bc = 12, 10, 2, "db2", "symmetric"
    plan = wl.Plan(h, w, J, filt, bc, "float64")
    blur = wl.Blur(h, w, 15, 3.0, dtype="float64")
    p = plan.p_valid
    Wm = O.synthesize(np.eye(p), h, w, J, filt, bc).reshape(p, h * w)
    RW = np.stack([O.blur(Wm[i].reshape(h, w)).ravel() for i in range(p)], 1)
    lmax = np.linalg.eigvalsh(RW.T @ RW).max()
    est = wl.lipschitz(plan, blur, iters=300, seed=3)
    assert est <= lmax * (1 + 1e-10)
    assert abs(est - lmax) <= 1e-8 * lmax


@pytest.mark.parametrize("filt,bc", [("cdf97", "symmetric"), ("db2", "periodic"), ("db4", "symmetric_edag"),
                                     ("db8", "zero")])
@pytest.mark.parametrize("dtype,tol", [("float64", 1e-13), ("float32", 2e-6)])
def test_fused_step_equals_grad_then_update(torch, filt, bc, dtype, tol):
    """wl_fista_step fuses the update into W*'s stores; it must equal wl_grad + wl_fista_update
    (and the oracle's step) from arbitrary (x, y), with the pitch padding left at 0."""
    h, w, J, B = 72, 56, 3, 2
    plan = wl.Plan(h, w, J, filt, bc, dtype)
    blur = wl.Blur(h, w, 15, 3.0, dtype=dtype)
    rng = np.random.default_rng(11)
    b = inputs.cast(rng.standard_normal((B, h, w)), dtype)
    x0, y0 = (inputs.cast(rng.standard_normal((B, plan.p_valid)), dtype) for _ in range(2))
    t, lam, lip = 3.0, 0.05, 1.3
    xd, yd = dev(torch, plan.from_packed(x0), dtype), dev(torch, plan.from_packed(y0), dtype)
    bd = dev(torch, b, dtype)
    g = wl.grad(plan, blur, yd, bd)
    xu, yu = xd.clone(), yd.clone()
    wl.fista_update(plan, g, xu, yu, t, lam, lip)
    wl.fista_step(plan, blur, bd, xd, yd, t, lam, lip)
    assert bool(torch.isfinite(xd).all()) and bool(torch.isfinite(yd).all())
    if dtype == "float64":
        assert float((xd - xu).abs().max()) <= 1e-13 * float(xu.abs().max())
        assert float((yd - yu).abs().max()) <= 1e-13 * float(yu.abs().max())
    go, _ = O.grad(y0.astype(np.float64), b.astype(np.float64), J, filt, bc)
    xo, yo, _ = O.fista_update(go, x0.astype(np.float64), y0.astype(np.float64), t, lam, lip)
    assert rel(plan.to_packed(xd.double().cpu().numpy()), xo) <= tol
    assert rel(plan.to_packed(yd.double().cpu().numpy()), yo) <= tol
    valid = np.zeros(plan.p_alloc, bool)
    valid[plan.to_packed(np.arange(plan.p_alloc)[None].astype(np.float64))[0].astype(np.int64)] = True
    assert np.all(xd.cpu().numpy()[:, ~valid] == 0) and np.all(yd.cpu().numpy()[:, ~valid] == 0)


@pytest.mark.parametrize("filt,bc", [("cdf97", "symmetric"), ("db4", "symmetric_edag"), ("haar", "symmetric")])
@pytest.mark.parametrize("dtype,tol", [("float64", 1e-12), ("float32", 2e-6)])
def test_pinv_gradient_matches_oracle(torch, filt, bc, dtype, tol):
    """wl_grad_adj(WL_ADJ_PINV): W-dagger closes the gradient."""
    h, w, J, B = 66, 50, 3, 2
    plan = wl.Plan(h, w, J, filt, bc, dtype)
    blur = wl.Blur(h, w, 15, 3.0, dtype=dtype)
    rng = np.random.default_rng(8)
    x = inputs.cast(rng.standard_normal((B, plan.p_valid)), dtype)
    b = inputs.cast(rng.standard_normal((B, h, w)), dtype)
    go, fo = O.grad(x.astype(np.float64), b.astype(np.float64), J, filt, bc, adjoint="pinv")
    f = torch.zeros(B, dtype=torch.float64, device="cuda")
    g = wl.grad(plan, blur, dev(torch, plan.from_packed(x), dtype), dev(torch, b, dtype), f=f, adjoint="pinv")
    assert rel(plan.to_packed(g.double().cpu().numpy()), go) <= tol
    np.testing.assert_allclose(f.cpu().numpy(), fo, rtol=tol)


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-11), ("float32", 1e-4)])
def test_fista_pinv_iterations_match_oracle(torch, dtype, tol):
    h, w, J, B, K, filt, bc = 40, 36, 3, 1, 10, "cdf97", "symmetric"
    plan = wl.Plan(h, w, J, filt, bc, dtype)
    blur = wl.Blur(h, w, 15, 3.0, dtype=dtype)
    rng = np.random.default_rng(6)
    b = inputs.cast(O.blur(inputs.blobs(rng, B, h, w, 8)) + 1e-3 * rng.standard_normal((B, h, w)), dtype)
    x, y, t, _ = O.fista(np.zeros((B, plan.p_valid)), b, J, filt, bc, 2e-3, 1.05, K, adjoint="pinv")
    xg, yg, tg = wl.fista(plan, blur, dev(torch, b, dtype), 2e-3, K, lip=1.05, adjoint="pinv")
    assert rel(plan.to_packed(xg.double().cpu().numpy()), x) <= tol
    assert rel(plan.to_packed(yg.double().cpu().numpy()), y) <= tol


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-12), ("float32", 1e-5)])
def test_fista_graph_replay_matches_eager(torch, dtype, tol):
    """Device-resident t + one captured iteration replayed (wl.fista(graph=True)) = the eager loop."""
    h, w, J, K = 48, 40, 3, 12
    plan = wl.Plan(h, w, J, "cdf97", "symmetric", dtype)
    blur = wl.Blur(h, w, 15, 3.0, dtype=dtype)
    rng = np.random.default_rng(21)
    b = dev(torch, inputs.cast(O.blur(inputs.blobs(rng, 2, h, w, 6)), dtype), dtype)
    xe, ye, te = wl.fista(plan, blur, b, 2e-3, K, lip=1.05)
    xg, yg, tg = wl.fista(plan, blur, b, 2e-3, K, lip=1.05, graph=True)
    assert tg == pytest.approx(te, rel=1e-14)
    assert float((xg - xe).abs().max()) <= tol * max(float(xe.abs().max()), 1e-30)
    assert float((yg - ye).abs().max()) <= tol * max(float(ye.abs().max()), 1e-30)


def test_cfg5_fused_fista_step_full_size(torch):
    """One fused FISTA step at the bench configuration (cfg5: 4 x 4096^2 CDF 9/7, 5 levels,
    symmetric, fp32), device-resident t, replayed as a CUDA graph like bench.py's FISTA line,
    against the oracle's grad + update."""
    c = inputs.CONFIGS[5]
    plan = wl.Plan(c.h, c.w, c.levels, c.filt, c.bc, c.dtype)
    blur = wl.Blur(c.h, c.w, inputs.BLUR_NTAPS, inputs.BLUR_SIGMA, dtype=c.dtype)
    x, y, bl, nz = inputs.workload(c, plan.p_valid)
    x = inputs.cast(x, c.dtype)
    y0 = inputs.cast(inputs.coefficients(np.random.default_rng(3), c.batch, plan.p_valid, 0.05), c.dtype)
    b = inputs.cast(O.blur(bl) + nz, c.dtype)
    xd = dev(torch, plan.from_packed(x), c.dtype)
    yd = dev(torch, plan.from_packed(y0), c.dtype)
    bd = dev(torch, b, c.dtype)
    t_dev = torch.full((1,), 2.0, dtype=torch.float64, device="cuda")
    ws = plan._ws(wl.OP_FISTA, c.batch, blur=blur)
    graph = wl.Graph(lambda: wl.fista_step(plan, blur, bd, xd, yd, t_dev, 1e-3, 1.1, ws=ws), warmup=0)
    graph.replay()
    torch.cuda.synchronize()
    g, _ = O.grad(y0.astype(np.float64), b.astype(np.float64), c.levels, c.filt, c.bc)
    xo, yo, to = O.fista_update(g, x.astype(np.float64), y0.astype(np.float64), 2.0, 1e-3, 1.1)
    assert float(t_dev.item()) == pytest.approx(to, rel=1e-15)
    assert rel(plan.to_packed(xd.double().cpu().numpy()), xo) <= 2e-6
    assert rel(plan.to_packed(yd.double().cpu().numpy()), yo) <= 2e-6
