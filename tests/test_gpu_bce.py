"""GPU Example 2 (blind channel estimation) against the fp64 oracle.

Tolerance: relative L2 error per output vector.  fp64 1e-12.  fp32: every output
is one dot product of length T (T = K for the convolution, N for S* r, C K for H* r) accumulated
in fp32 FMAs; with random-sign terms the rounding error grows like eps32 sqrt(T) relative to the
result, so the bound is 4 eps32 sqrt(T_max) = 2e-5 at the paper's sizes (T = 1767), held to 2e-5.
"""
import numpy as np
import pytest

from oracle import bce as OB
from paper_1707_02018_b200 import inputs, wl

pytestmark = pytest.mark.gpu

SIZES = [(1, 1), (1, 7), (6, 1), (3, 5), (13, 29), (17, 40), (64, 33), (130, 9), (844, 1767), (894, 1717)]
TOL = {"float64": 1e-12, "float32": 2e-5}


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def dev(torch, a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=getattr(torch, dtype))


def rel_rows(a, b):
    a = a.reshape(-1, a.shape[-1])
    b = b.reshape(-1, b.shape[-1])
    return float(np.max(np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-300)))


@pytest.mark.parametrize("K,N", SIZES)
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_conv_and_adjoints(torch, K, N, dtype):
    rng = np.random.default_rng(K * 7919 + N)
    B = 3
    h = inputs.cast(rng.standard_normal((B, K)), dtype)
    s = inputs.cast(rng.standard_normal((B, N)), dtype)
    r = inputs.cast(rng.standard_normal((B, K + N - 1)), dtype)
    hd, sd, rd = dev(torch, h, dtype), dev(torch, s, dtype), dev(torch, r, dtype)
    x = wl.conv_full(hd, sd)
    gh = wl.conv_adjoint_h(sd, rd, K)
    gs = wl.conv_adjoint_s(hd, rd, N)
    torch.cuda.synchronize()
    assert rel_rows(x.double().cpu().numpy(), OB.conv_full(h, s)) <= TOL[dtype]
    assert rel_rows(gh.double().cpu().numpy(), OB.conv_adjoint_h(s, r, K)) <= TOL[dtype]
    assert rel_rows(gs.double().cpu().numpy(), OB.conv_adjoint_s(h, r, N)) <= TOL[dtype]


def test_conv_adjoint_identity_fp64(torch):
    """<S h, r> = <h, S* r> and <H s, r> = <s, H* r> on the GPU results (fp64 host inner products)."""
    rng = np.random.default_rng(4)
    K, N, B = 844, 1767, 4
    h, s, r = rng.standard_normal((B, K)), rng.standard_normal((B, N)), rng.standard_normal((B, K + N - 1))
    hd, sd, rd = (dev(torch, a, "float64") for a in (h, s, r))
    x = wl.conv_full(hd, sd).cpu().numpy()
    gh = wl.conv_adjoint_h(sd, rd, K).cpu().numpy()
    gs = wl.conv_adjoint_s(hd, rd, N).cpu().numpy()
    lhs = np.sum(x * r, -1)
    assert np.allclose(lhs, np.sum(h * gh, -1), rtol=1e-12)
    assert np.allclose(lhs, np.sum(s * gs, -1), rtol=1e-12)


@pytest.mark.parametrize("P,C,K,N,shared", [(3, 2, 5, 9, False), (2, 1, 1, 1, False), (4, 3, 37, 61, True),
                                            (2, 2, 844, 1767, True), (2, 2, 894, 1717, False)])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_bce_grad_matches_oracle(torch, P, C, K, N, shared, dtype):
    rng = np.random.default_rng(P * 1000 + K)
    h = inputs.cast(rng.standard_normal((P, C, K)), dtype)
    s = inputs.cast(rng.standard_normal((P, N)), dtype)
    x = inputs.cast(rng.standard_normal((C, K + N - 1) if shared else (P, C, K + N - 1)), dtype)
    lam, delta = 0.3, 0.4
    F, gh_o, gs_o = OB.bce_smooth(h, s, x if not shared else np.broadcast_to(x, (P,) + x.shape), lam, delta)
    f = torch.zeros(P, dtype=torch.float64, device="cuda")
    gh, gs = wl.bce_grad(dev(torch, h, dtype), dev(torch, s, dtype), dev(torch, x, dtype), lam, delta, f=f)
    assert rel_rows(gh.double().cpu().numpy(), gh_o) <= TOL[dtype]
    assert rel_rows(gs.double().cpu().numpy(), gs_o) <= TOL[dtype]
    np.testing.assert_allclose(f.cpu().numpy(), F, rtol=TOL[dtype])


def test_bce_grad_paper_workload_sampled(torch):
    """Paper sizes (two channels, K_est = 844, N_est = 1767) with 256 random starts against
    one shared synthetic observation; a sample of problems is checked against the oracle."""
    c = inputs.BCE
    P = 256
    ht, st, nz, h0, s0 = inputs.bce_problem(11, P, c["channels"], c["K"], c["N"], c["K_est"], c["N_est"], c["noise"])
    x = np.stack([np.convolve(ht[i], st) for i in range(c["channels"])]) + nz
    h32, s32, x32 = (inputs.cast(a, "float32") for a in (h0, s0, x))
    f = torch.zeros(P, dtype=torch.float64, device="cuda")
    gh, gs = wl.bce_grad(dev(torch, h32, "float32"), dev(torch, s32, "float32"), dev(torch, x32, "float32"),
                         c["lam_tv"], c["delta"], f=f)
    gh, gs, f = gh.double().cpu().numpy(), gs.double().cpu().numpy(), f.cpu().numpy()
    for p in (0, 1, 97, 255):
        F, gho, gso = OB.bce_smooth(h32[p], s32[p], x32, c["lam_tv"], c["delta"])
        assert rel_rows(gh[p], gho) <= TOL["float32"]
        assert rel_rows(gs[p], gso) <= TOL["float32"]
        assert abs(f[p] - F) <= TOL["float32"] * F


def test_bce_zero_gradient_at_noiseless_solution(torch):
    rng = np.random.default_rng(9)
    C, K, N = 2, 40, 70
    h, s = rng.standard_normal((1, C, K)), rng.standard_normal((1, N))
    x = np.stack([np.convolve(h[0, i], s[0]) for i in range(C)])[None]
    gh, gs = wl.bce_grad(dev(torch, h, "float64"), dev(torch, s, "float64"), dev(torch, x, "float64"), 0.0, 0.1)
    assert float(gh.abs().max()) < 1e-11 and float(gs.abs().max()) < 1e-11


def test_bce_errors(torch):
    h = torch.zeros(1, 2, 5, device="cuda")
    s = torch.zeros(1, 9, device="cuda")
    x = torch.zeros(2, 13, device="cuda")
    with pytest.raises(wl.WLError):
        wl.bce_grad(h, s, x, 0.01, 0.0)                 # delta must be > 0
    with pytest.raises(wl.WLError):
        big = torch.zeros(1, 2, 20000, device="cuda")
        wl.bce_grad(big, torch.zeros(1, 20000, device="cuda"), torch.zeros(2, 39999, device="cuda"))  # smem
    with pytest.raises(ValueError):
        wl.bce_grad(h, s, torch.zeros(2, 12, device="cuda"))
