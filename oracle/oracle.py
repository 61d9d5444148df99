"""Python face of the fp64 CPU oracle.  TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / reference
leg may import this module.  The arithmetic lives in `oracle/oracle.c` (plain fp64
loops) and `oracle/filters.py` (filter construction); this file only chooses which
filters / extension / fold each operator uses -- the readings of the paper listed
in DESIGN.md "Readings" -- and marshals numpy arrays.

Operators (PAPER.md §"Example 1: An Image Deblurring Problem"):
  analyze    W-dagger = W-dagger_zpd E_bc
  adjoint    W*       = W~dagger_zpd (E^dagger)*                    (Eq. (4))
  synthesize W        = (W*)^T                                      (reading R1)
  analyze_adjoint (W-dagger)* = E_bc^T A_a^T
  blur       R        (Gaussian PSF, symmetric BC)
  blur_adjoint R*
  grad       grad f(x) = W* R* (R W x - b),  f = 1/2 ||R W x - b||^2
Reading R1 ("C", the toolbox-consistent pair): for bc in {zero, symmetric} W* uses
E_zpd and W crops; for periodic both use the periodisation wrap; the paper-literal
symmetric variant "symmetric_edag" uses (E_sym^dagger)* = E_sym diag(1/c) and its
transpose (Eq. (4)).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from .filters import filter_bank, gaussian_taps

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

EXT_ZERO, EXT_PER, EXT_SYM, EXT_SYM_PADJ = 0, 1, 2, 3
FOLD_CROP, FOLD_WRAP, FOLD_SYM_PINV, FOLD_SYM_T = 0, 1, 2, 3

BCS = ("zero", "periodic", "symmetric", "symmetric_edag")

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, no fast-math, OpenMP)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off",
                               "-fopenmp", "-shared", "-fPIC", src, "-o", _LIB_PATH, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        lp = ctypes.POINTER(ctypes.c_long)
        cl, ci = ctypes.c_long, ctypes.c_int
        L.wlo_extend1d.argtypes = [dp, cl, cl, ci, ci, dp]
        L.wlo_extend_adjoint1d.argtypes = [dp, cl, cl, ci, ci, dp]
        L.wlo_chain.argtypes = [cl, ci, ci, ci, lp]
        L.wlo_num_coeffs.argtypes = [cl, cl, ci, ci, ci]
        L.wlo_num_coeffs.restype = cl
        L.wlo_analysis2d.argtypes = [dp, cl, cl, cl, ci, dp, dp, ci, ci, dp]
        L.wlo_synthesis2d.argtypes = [dp, cl, cl, cl, ci, dp, dp, ci, ci, dp]
        L.wlo_blur2d.argtypes = [dp, cl, cl, cl, dp, ci, ci, dp]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ extension
_KIND = {"zero": EXT_ZERO, "periodic": EXT_PER, "symmetric": EXT_SYM}


def extend(y, Lp: int, kind: str) -> np.ndarray:
    """E y over t in [-Lp, n+Lp)."""
    y = _f64(y)
    out = np.empty(y.size + 2 * Lp)
    lib().wlo_extend1d(_dp(y), y.size, Lp, _KIND[kind], 0, _dp(out))
    return out


def extend_pinv_adjoint(y, Lp: int, kind: str) -> np.ndarray:
    """(E^dagger)* y = E diag(1/c) y."""
    y = _f64(y)
    out = np.empty(y.size + 2 * Lp)
    lib().wlo_extend1d(_dp(y), y.size, Lp, _KIND[kind], 1, _dp(out))
    return out


def extend_adjoint(v, n: int, Lp: int, kind: str, pinv: bool = False) -> np.ndarray:
    """E^T v (pinv=False) or E^dagger v (pinv=True)."""
    v = _f64(v)
    assert v.size == n + 2 * Lp
    out = np.empty(n)
    lib().wlo_extend_adjoint1d(_dp(v), n, Lp, _KIND[kind], int(pinv), _dp(out))
    return out


# --------------------------------------------------------------- level chain
def chain(n: int, L: int, bc: str, J: int):
    """[n_0, ..., n_J] with n_j = floor((n_{j-1}+L-1)/2) (zero/sym) or n_{j-1}/2 (per)."""
    kind = EXT_PER if bc == "periodic" else (EXT_SYM if bc.startswith("symmetric") else EXT_ZERO)
    out = (ctypes.c_long * (J + 1))()
    rc = lib().wlo_chain(n, L, kind, J, out)
    if rc != 0:
        raise ValueError(f"level {-rc} cannot be formed from length chain starting at {n} (bc={bc}, L={L})")
    return [int(v) for v in out]


@dataclass(frozen=True)
class Layout:
    """Oracle packed coefficient layout: LL_J, then (LH_j, HL_j, HH_j) for j = J..1."""
    h: int
    w: int
    J: int
    c0: tuple
    c1: tuple

    @property
    def p(self) -> int:
        return self.c0[self.J] * self.c1[self.J] + sum(3 * self.c0[j] * self.c1[j] for j in range(1, self.J + 1))

    def bands(self):
        """List of (name, level, offset, rows, cols) in packing order."""
        out = [("LL", self.J, 0, self.c0[self.J], self.c1[self.J])]
        off = self.c0[self.J] * self.c1[self.J]
        for j in range(self.J, 0, -1):
            for nm in ("LH", "HL", "HH"):
                out.append((nm, j, off, self.c0[j], self.c1[j]))
                off += self.c0[j] * self.c1[j]
        return out


def layout(h: int, w: int, J: int, filt: str, bc: str) -> Layout:
    L = filter_bank(filt).L
    return Layout(h, w, J, tuple(chain(h, L, bc, J)), tuple(chain(w, L, bc, J)))


# ----------------------------------------------------------------- operators
def _batch(a, trailing):
    a = _f64(a)
    if a.ndim == trailing:
        return a[None], True
    return a, False


def _analysis(img, J, flo, fhi, L, ext):
    img, squeeze = _batch(img, 2)
    B, h, w = img.shape
    p = lib().wlo_num_coeffs(h, w, L, ext, J)
    if p < 0:
        raise ValueError("invalid level chain")
    x = np.empty((B, p))
    rc = lib().wlo_analysis2d(_dp(img), B, h, w, J, _dp(_f64(flo)), _dp(_f64(fhi)), L, ext, _dp(x))
    assert rc == 0, rc
    return x[0] if squeeze else x


def _synthesis(x, h, w, J, glo, ghi, L, fold):
    x, squeeze = _batch(x, 1)
    B = x.shape[0]
    img = np.empty((B, h, w))
    rc = lib().wlo_synthesis2d(_dp(x), B, h, w, J, _dp(_f64(glo)), _dp(_f64(ghi)), L, fold, _dp(img))
    assert rc == 0, rc
    return img[0] if squeeze else img


def analyze(img, J: int, filt: str, bc: str) -> np.ndarray:
    """W-dagger: analysis filters over E_bc."""
    fb = filter_bank(filt)
    ext = {"zero": EXT_ZERO, "periodic": EXT_PER, "symmetric": EXT_SYM, "symmetric_edag": EXT_SYM}[bc]
    return _analysis(img, J, fb.a_lo, fb.a_hi, fb.L, ext)


def adjoint(img, J: int, filt: str, bc: str) -> np.ndarray:
    """W*: dual filters over (E^dagger)* (Eq. (4); reading R1)."""
    fb = filter_bank(filt)
    ext = {"zero": EXT_ZERO, "periodic": EXT_PER, "symmetric": EXT_ZERO, "symmetric_edag": EXT_SYM_PADJ}[bc]
    return _analysis(img, J, fb.d_lo, fb.d_hi, fb.L, ext)


_adjoint_op = adjoint  # grad's `adjoint` argument shadows the name


def synthesize(x, h: int, w: int, J: int, filt: str, bc: str) -> np.ndarray:
    """W = (W*)^T: scatter with the dual filters, then the fold adjoint to W*'s extension."""
    fb = filter_bank(filt)
    fold = {"zero": FOLD_CROP, "periodic": FOLD_WRAP, "symmetric": FOLD_CROP, "symmetric_edag": FOLD_SYM_PINV}[bc]
    return _synthesis(x, h, w, J, fb.d_lo, fb.d_hi, fb.L, fold)


def analyze_adjoint(x, h: int, w: int, J: int, filt: str, bc: str) -> np.ndarray:
    """(W-dagger)*: the adjoint of the analysis W-dagger = A_a E_bc ("(and analysis)";
    SURVEY §8(f) NEXT #2): scatter with the ANALYSIS filters, then fold with E_bc^T --
    truncate (zero), wrap-add (periodic), reflect-add (symmetric, symmetric_edag)."""
    fb = filter_bank(filt)
    fold = {"zero": FOLD_CROP, "periodic": FOLD_WRAP, "symmetric": FOLD_SYM_T, "symmetric_edag": FOLD_SYM_T}[bc]
    return _synthesis(x, h, w, J, fb.a_lo, fb.a_hi, fb.L, fold)


def blur(img, taps=None) -> np.ndarray:
    """R: per axis crop o conv o E_sym, separable (reading R12)."""
    taps = gaussian_taps() if taps is None else _f64(taps)
    img, squeeze = _batch(img, 2)
    out = np.empty_like(img)
    rc = lib().wlo_blur2d(_dp(img), img.shape[0], img.shape[1], img.shape[2], _dp(taps), taps.size, 0, _dp(out))
    assert rc == 0
    return out[0] if squeeze else out


def blur_adjoint(img, taps=None) -> np.ndarray:
    """R*: per axis E_sym^T o full correlation (reflect-add), separable."""
    taps = gaussian_taps() if taps is None else _f64(taps)
    img, squeeze = _batch(img, 2)
    out = np.empty_like(img)
    rc = lib().wlo_blur2d(_dp(img), img.shape[0], img.shape[1], img.shape[2], _dp(taps), taps.size, 1, _dp(out))
    assert rc == 0
    return out[0] if squeeze else out


def grad(x, b, J: int, filt: str, bc: str, taps=None, adjoint: str = "true"):
    """grad f(x) = W* R* (R W x - b) and f = 1/2 ||R W x - b||^2 per image.

    Evaluated literally, in that order, in fp64.  adjoint="pinv" replaces W* by W-dagger, the
    approximation W* ~ W-dagger that P:113-117 and P:176-177 run FISTA with.
    """
    b = _f64(b)
    h, w = b.shape[-2:]
    u = synthesize(x, h, w, J, filt, bc)
    r = blur(u, taps) - b
    s = blur_adjoint(r, taps)
    g = _adjoint_op(s, J, filt, bc) if adjoint == "true" else analyze(s, J, filt, bc)
    f = 0.5 * np.sum(r.reshape(r.shape[:-2] + (-1,)) ** 2, axis=-1)
    return g, f


# ------------------------------------------------- FISTA: SURVEY §8(f) NEXT #1
def soft_threshold(v, tau):
    """prox of tau ||.||_1: sign(v) max(|v| - tau, 0)."""
    return np.sign(v) * np.maximum(np.abs(v) - tau, 0.0)


def fista_update(g, x, y, t, lam, lip):
    """One FISTA update (Beck & Teboulle 2009, cited at P:117) from g = grad f(y):
        x+ = soft(y - g / L, lam / L);  t+ = (1 + sqrt(1 + 4 t^2)) / 2;  y+ = x+ + ((t - 1) / t+)(x+ - x).
    Returns (x+, y+, t+)."""
    x_new = soft_threshold(y - g / lip, lam / lip)
    t_new = (1.0 + np.sqrt(1.0 + 4.0 * t * t)) / 2.0
    y_new = x_new + ((t - 1.0) / t_new) * (x_new - x)
    return x_new, y_new, t_new


def fista(x0, b, J: int, filt: str, bc: str, lam: float, lip: float, iters: int, taps=None, adjoint: str = "true"):
    """FISTA on min_x 1/2 ||R W x - b||^2 + lam ||x||_1 (Eq. (1)): `iters` steps from x0,
    y_1 = x0, t_1 = 1.  Returns (x, y, t, objective trace F(x_k))."""
    x = np.array(x0, dtype=np.float64)
    y = x.copy()
    t = 1.0
    trace = []
    for _ in range(iters):
        g, _f = grad(y, b, J, filt, bc, taps, adjoint)
        x, y, t = fista_update(g, x, y, t, lam, lip)
        _g, fx = grad(x, b, J, filt, bc, taps)
        trace.append(fx + lam * np.abs(x).reshape(x.shape[0] if x.ndim > 1 else 1, -1).sum(axis=-1))
    return x, y, t, np.array(trace)


def lipschitz(v0, h: int, w: int, J: int, filt: str, bc: str, iters: int, taps=None):
    """Power iteration for L = lambda_max(W* R* R W) (the Lipschitz constant of grad f):
    v <- G v / ||G v|| with G v = grad f(v) at b = 0; returns the Rayleigh quotient <v, G v> / <v, v>
    of the last iterate (a lower bound of L that increases to it)."""
    v = np.array(v0, dtype=np.float64).reshape(1, -1)
    zero = np.zeros((1, h, w))
    est = 0.0
    for _ in range(iters):
        v = v / np.linalg.norm(v)
        gv, _f = grad(v, zero, J, filt, bc, taps)
        est = float(np.vdot(v, gv))
        v = gv
    return est
