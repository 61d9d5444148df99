"""GPU parity of the register-ring blur kernels (`k_blur_ring`, fp32, PSFs of 3..15 taps) against
the fp64 oracle's R, R* and R*(R u - b) (reading R12).

The shapes drive every path of the kernel: several strips with a ragged last strip (the residual
strip is 256 - 2h output columns wide, R's 256), widths smaller than one strip, images shorter
than one row group (5 rows) or than the PSF window, many row bands per strip (a single tall
image), top / bottom groups gathered with reflected rows, and left / right columns read
mirrored.  Both the relative L2 error (BASELINE.json bar) and an elementwise bound are checked.
"""
import numpy as np
import pytest

from oracle import oracle as O
from oracle.filters import gaussian_taps
from paper_1707_02018_b200 import inputs, wl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    return t.detach().double().cpu().numpy()


def check(got, want, what):
    B = want.shape[0]
    g, r = got.reshape(B, -1), want.reshape(B, -1)
    rel = np.max(np.linalg.norm(g - r, axis=1) / np.maximum(np.linalg.norm(r, axis=1), 1e-300))
    assert rel <= 2e-6, f"{what}: relative L2 {rel:.3e}"
    # elementwise: every output is a short sum of terms bounded by max|input|
    err = np.abs(g - r).max(axis=1)
    scale = np.maximum(np.abs(r).max(axis=1), 1e-30)
    assert np.all(err <= 4e-6 * scale), f"{what}: max elementwise error {np.max(err / scale):.3e} of max|ref|"


SHAPES = [(1, 64, 520), (2, 37, 244), (1, 300, 1000), (3, 5, 16), (2, 3, 12), (1, 1100, 24),
          (2, 17, 260), (1, 8, 4)]


@pytest.mark.parametrize("ntaps", [15, 3, 9, 13])
@pytest.mark.parametrize("B,h,w", SHAPES)
def test_ring_blur_and_residual(torch, ntaps, B, h, w):
    hw = ntaps // 2
    if h < hw or w < hw:
        pytest.skip("blur plans need h, w >= ntaps/2")
    taps = gaussian_taps(ntaps, 3.0 if ntaps == 15 else 2.0)
    blur = wl.Blur(h, w, taps=taps, dtype="float32")
    rng = np.random.default_rng(ntaps * 1000 + h + w)
    u = inputs.cast(rng.standard_normal((B, h, w)), "float32")
    b = inputs.cast(rng.standard_normal((B, h, w)), "float32")
    ud, bd = dev(torch, u), dev(torch, b)
    check(host(blur.apply(ud)), O.blur(u, taps), "R")
    check(host(blur.adjoint(ud)), O.blur_adjoint(u, taps), "R*")
    f = torch.zeros(B, dtype=torch.float64, device="cuda")
    s = host(blur.residual_adjoint(ud, bd, f=f))
    r = O.blur(u, taps) - b
    check(s, O.blur_adjoint(r, taps), "R*(Ru - b)")
    fref = 0.5 * np.sum(r.reshape(B, -1) ** 2, axis=1)
    np.testing.assert_allclose(host(f), fref, rtol=1e-5)
    # without f the outputs are the same
    s2 = host(blur.residual_adjoint(ud, bd))
    np.testing.assert_array_equal(s2, s)


def test_ring_residual_cfg5_full_images(torch):
    """cfg5 shape (4 x 4096^2, 15 taps, sigma 3) in the launch configuration the bench times;
    images 0 and 3 compared in full with the oracle (about 3 s of fp64 CPU work each)."""
    B, h, w = 4, 4096, 4096
    blur = wl.Blur(h, w, 15, 3.0, dtype="float32")
    rng = np.random.default_rng(5)
    ud = dev(torch, inputs.cast(rng.standard_normal((B, h, w)), "float32"))
    bd = dev(torch, inputs.cast(rng.standard_normal((B, h, w)), "float32"))
    f = torch.zeros(B, dtype=torch.float64, device="cuda")
    s = blur.residual_adjoint(ud, bd, f=f)
    for img in (0, 3):
        u = host(ud[img:img + 1])
        r = O.blur(u) - host(bd[img:img + 1])
        check(host(s[img:img + 1]), O.blur_adjoint(r), f"cfg5 image {img}")
        np.testing.assert_allclose(host(f)[img], 0.5 * np.sum(r ** 2), rtol=1e-5)
