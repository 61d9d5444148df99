"""CPU-side checks of libwl: it loads, exports every symbol include/wl.h declares, and its
host logic (level chains, subband table, filters, validation) agrees with the oracle.
No compute call is made here (there is no GPU in this tier)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1707_02018_b200 import inputs, wl
from oracle import oracle as O
from oracle.filters import FILTERS, filter_bank, gaussian_taps

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "wl.h")).read()
    return sorted(set(re.findall(r"WL_API\s+[\w\s\*]*?\b(wl_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = wl.lib()
    syms = declared_symbols()
    assert len(syms) >= 19
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(wl.EXPORTS)
    assert b"sm_100a" in L.wl_version()


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", os.path.join(ROOT, "paper_1707_02018_b200",
                                                                                   "libwl.so")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("cfg", sorted(inputs.CONFIGS))
def test_plan_matches_oracle_layout(cfg):
    c = inputs.CONFIGS[cfg]
    p = wl.Plan(c.h, c.w, c.levels, c.filt, c.bc, c.dtype)
    lay = O.layout(c.h, c.w, c.levels, c.filt, c.bc)
    assert p.chain_h == list(lay.c0) and p.chain_w == list(lay.c1)
    assert p.p_valid == lay.p
    ob = lay.bands()
    assert [(b.name, b.level, b.rows, b.cols) for b in p.bands] == [(n, j, r, cc) for n, j, _, r, cc in ob]
    es = 8 if c.dtype == "float64" else 4
    for b in p.bands:
        assert b.pitch >= b.cols and (b.pitch * es) % 16 == 0 and (b.offset * es) % 16 == 0
    # layout helpers round-trip
    xp = np.arange(p.p_valid, dtype=np.float64)
    np.testing.assert_array_equal(p.to_packed(p.from_packed(xp)), xp)


@pytest.mark.parametrize("filt", FILTERS)
def test_library_filters_match_oracle(filt):
    p = wl.Plan(64, 64, 1, filt, "zero", "float64")
    fb = filter_bank(filt)
    for got, ref in zip(p.filters(), (fb.a_lo, fb.a_hi, fb.d_lo, fb.d_hi)):
        np.testing.assert_allclose(got, ref, rtol=0, atol=2e-15)


def test_library_gaussian_taps_match_oracle():
    b = wl.Blur(64, 64, 15, 3.0)
    np.testing.assert_allclose(b.taps(), gaussian_taps(15, 3.0), rtol=0, atol=1e-16)


@pytest.mark.parametrize("h,w,J,filt,bc", [(20, 20, 3, "db2", "periodic"), (10, 40, 1, "db8", "symmetric"),
                                            (0, 5, 1, "haar", "zero"), (16, 16, 33, "haar", "zero"),
                                            (16, 16, 0, "haar", "zero")])
def test_plan_rejects_impossible_sizes(h, w, J, filt, bc):
    with pytest.raises(wl.WLError) as ei:
        wl.Plan(h, w, J, filt, bc)
    assert ei.value.status == wl.WL_ESIZE
    if J in (1, 3) and h > 0:
        assert "level" in str(ei.value)


def test_plan_accepts_saturating_symmetric_chain():
    p = wl.Plan(15, 40, 6, "db8", "symmetric", "float32")      # floor((15+15)/2) = 15: fixed point
    assert p.chain_h == [15] * 7


def test_plan_rejects_unknown_enums():
    L = wl.lib()
    h = ctypes.c_void_p()
    assert L.wl_plan_create(ctypes.byref(h), 16, 16, 1, 3, 0, 0) == wl.WL_EINVAL      # filter 3
    assert L.wl_plan_create(ctypes.byref(h), 16, 16, 1, 2, 7, 0) == wl.WL_EINVAL      # bc 7
    assert L.wl_plan_create(ctypes.byref(h), 16, 16, 1, 2, 0, 5) == wl.WL_EINVAL      # dtype 5
    assert b"dtype" in L.wl_last_error()


def test_blur_rejects_bad_taps():
    with pytest.raises(wl.WLError):
        wl.Blur(32, 32, taps=[0.2, 0.5, 0.3])          # not symmetric: R* != R
    with pytest.raises(wl.WLError):
        wl.Blur(32, 32, taps=[0.5, 0.5])               # even length
    with pytest.raises(wl.WLError):
        wl.Blur(5, 32, ntaps=15)                        # h < ntaps/2


def test_workspace_bytes():
    p = wl.Plan(4096, 4096, 5, "cdf97", "symmetric", "float32")
    b = wl.Blur(4096, 4096)
    n_adj = p.workspace_bytes(wl.OP_ADJOINT, 4)
    n_grad = p.workspace_bytes(wl.OP_GRAD, 4, b)
    assert n_adj >= 4 * 2052 * 2052 * 4            # LL_1 of every image
    assert n_grad >= n_adj + 2 * 4 * 4096 * 4096 * 4
    assert p.workspace_bytes(wl.OP_ADJOINT, 0) == 0
    single = wl.Plan(64, 64, 1, "haar", "zero", "float32")
    assert single.workspace_bytes(wl.OP_ADJOINT, 3) == 0     # J = 1: no intermediate LL


def test_compute_calls_refuse_cpu_tensors():
    torch = pytest.importorskip("torch")
    p = wl.Plan(32, 32, 2, "db2", "zero", "float32")
    with pytest.raises(ValueError):
        p.adjoint(torch.zeros(32, 32))


def test_new_entry_points_validate_before_any_launch():
    """The FISTA / host-buffer / adjoint-choice / Example 2 entry points reject bad arguments with a
    status and a message before touching the device (so this runs without a GPU)."""
    L = wl.lib()
    p = wl.Plan(32, 32, 2, "db2", "symmetric", "float32")
    b = wl.Blur(32, 32)
    bad_blur = wl.Blur(32, 40)
    vp = ctypes.c_void_p
    assert L.wl_grad_adj(p._h, b._h, 1, vp(16), vp(32), vp(48), None, 7, None, None) == wl.WL_EINVAL
    assert b"adj" in L.wl_last_error()
    assert L.wl_grad_host(p._h, None, 1, vp(16), vp(32), vp(48), None, None, None) == wl.WL_EINVAL
    assert L.wl_grad_host(p._h, bad_blur._h, 1, vp(16), vp(32), vp(48), None, None, None) == wl.WL_EINVAL
    assert L.wl_grad_host(p._h, b._h, 1, None, vp(32), vp(48), None, None, None) == wl.WL_EINVAL
    assert L.wl_grad_host(p._h, b._h, 0, None, None, None, None, None, None) == wl.WL_OK   # empty batch
    assert L.wl_fista_step_dev(p._h, b._h, 1, vp(16), vp(32), vp(48), None, 0.1, 1.0, None, 0, None,
                               None) == wl.WL_EINVAL
    assert b"t_dev" in L.wl_last_error()
    assert L.wl_fista_step(p._h, b._h, 1, vp(16), vp(32), vp(48), 0.5, 0.1, 1.0, None, 0, None, None,
                           None) == wl.WL_EINVAL                                            # t < 1
    assert L.wl_fista_update(p._h, 1, vp(16), vp(32), vp(48), 1.0, 0.1, 0.0, None, None) == wl.WL_EINVAL  # lip = 0
    # t_{k+1} comes back through the host out-pointer (batch 0: no launch, no device pointer needed)
    tn = ctypes.c_double()
    assert L.wl_fista_update(p._h, 0, None, None, None, 1.0, 0.1, 1.0, ctypes.byref(tn), None) == wl.WL_OK
    assert tn.value == (1.0 + 5.0 ** 0.5) / 2.0
    tn2 = ctypes.c_double()
    assert L.wl_fista_step(p._h, b._h, 0, None, None, None, tn.value, 0.1, 1.0, None, 0, None, ctypes.byref(tn2),
                           None) == wl.WL_OK
    assert abs(tn2.value - (1.0 + (1.0 + 4.0 * tn.value ** 2) ** 0.5) / 2.0) < 1e-15
    # Example 2
    assert L.wl_bce_grad(0, 1, 2, 5, 9, vp(16), vp(32), vp(48), 0, 0.01, 0.0, vp(64), vp(80), None,
                         None) == wl.WL_EINVAL                                              # delta = 0
    assert L.wl_bce_grad(0, 1, 0, 5, 9, vp(16), vp(32), vp(48), 0, 0.01, 0.1, vp(64), vp(80), None,
                         None) == wl.WL_EINVAL                                              # channels = 0
    assert L.wl_bce_grad(0, 1, 2, 20000, 20000, vp(16), vp(32), vp(48), 0, 0.01, 0.1, vp(64), vp(80), None,
                         None) == wl.WL_ESIZE                                               # shared memory
    assert L.wl_conv_full(0, 1, 0, 9, vp(16), vp(32), vp(48), None) == wl.WL_ESIZE       # K = 0
    assert L.wl_conv_full(5, 1, 3, 9, vp(16), vp(32), vp(48), None) == wl.WL_EDTYPE      # bad dtype
    assert L.wl_conv_adjoint_h(0, 0, 3, 9, None, None, None, None) == wl.WL_OK           # empty batch


def test_binding_batch_helpers():
    """The binding's batch / f checks: pure metadata logic, checked on CPU tensors."""
    import torch
    wl._same_batch(4, (torch.zeros(4, 10), "x", 1), (torch.zeros(2, 2, 3, 3), "b", 2), (None, "f", 1))
    with pytest.raises(ValueError, match="batch 1"):
        wl._same_batch(4, (torch.zeros(1, 10), "b", 1))
    with pytest.raises(ValueError, match="batch 3"):
        wl._same_batch(1, (torch.zeros(3, 5, 5), "img", 2))
    wl._same_batch(1, (torch.zeros(5, 5), "img", 2))              # no leading dims = batch 1
