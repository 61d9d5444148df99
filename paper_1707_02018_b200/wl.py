"""Thin Python binding of libwl (include/wl.h) -- argument marshalling only.

Every step of every operator runs in the CUDA kernels of libwl.so; this module only
checks tensor metadata, allocates outputs / workspace with torch (device memory is
plumbing) and passes raw pointers plus the current CUDA stream through ctypes.
There is no CPU fallback: if libwl.so cannot be loaded, or a tensor is not on a CUDA
device, the call raises.

Names follow the paper: W = synthesize, W* = adjoint, W-dagger = analyze,
R = blur, R* = blur_adjoint, grad f = W* R* (R W x - b).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("WL_LIB") or os.path.join(_PKG, "libwl.so")   # WL_LIB: A/B builds (tools)

WL_OK, WL_EINVAL, WL_ESIZE, WL_EDTYPE, WL_EALIGN, WL_ENOMEM, WL_ECUDA = range(7)
FILTERS = {"haar": 1, "db1": 1, "db2": 2, "db4": 4, "db8": 8, "cdf97": 97}
BCS = {"zero": 0, "periodic": 1, "symmetric": 2, "symmetric_edag": 3}
OP_SYNTHESIZE, OP_ADJOINT, OP_ANALYZE, OP_GRAD, OP_ANALYZE_ADJOINT, OP_FISTA, OP_LIPSCHITZ, OP_GRAD_HOST = range(8)
MAX_LEVELS = 32


class WLError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"wl status {status}: {msg}")
        self.status = status


class _Subband(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_int64), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("pitch", ctypes.c_int64)]


class _PlanInfo(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int), ("filter_length", ctypes.c_int), ("p_valid", ctypes.c_int64),
                ("p_alloc", ctypes.c_int64), ("h", ctypes.c_int64 * (MAX_LEVELS + 1)),
                ("w", ctypes.c_int64 * (MAX_LEVELS + 1)), ("band", _Subband * (1 + 3 * MAX_LEVELS))]


EXPORTS = ("wl_plan_create", "wl_plan_destroy", "wl_plan_query", "wl_plan_filters", "wl_workspace_bytes",
           "wl_synthesize", "wl_adjoint", "wl_analyze", "wl_analyze_adjoint", "wl_blur_create", "wl_blur_create_gaussian",
           "wl_blur_destroy", "wl_blur_taps", "wl_blur", "wl_blur_adjoint", "wl_blur_residual_adjoint",
           "wl_grad", "wl_grad_host", "wl_grad_adj", "wl_fista_update", "wl_fista_step", "wl_fista_step_dev", "wl_lipschitz", "wl_conv_full", "wl_conv_adjoint_h",
           "wl_conv_adjoint_s", "wl_bce_grad", "wl_last_error", "wl_launch_count",
           "wl_version")

_lib = None


def lib():
    """Load libwl.so (built in-tree by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        if os.path.exists("/usr/local/cuda/bin/nvcc") or os.environ.get("NVCC"):
            from ._build import build
            build()
        else:
            raise ImportError(f"{_LIB_PATH} is missing; run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(_LIB_PATH)
    vp, i64, ci, cd = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    dp = ctypes.POINTER(ctypes.c_double)
    L.wl_plan_create.argtypes = [ctypes.POINTER(vp), i64, i64, ci, ci, ci, ci]
    L.wl_plan_destroy.argtypes = [vp]
    L.wl_plan_destroy.restype = None
    L.wl_plan_query.argtypes = [vp, ctypes.POINTER(_PlanInfo)]
    L.wl_plan_filters.argtypes = [vp, dp, dp, dp, dp]
    L.wl_workspace_bytes.argtypes = [vp, vp, ci, i64]
    L.wl_workspace_bytes.restype = ctypes.c_size_t
    for fn in ("wl_synthesize", "wl_adjoint", "wl_analyze", "wl_analyze_adjoint"):
        getattr(L, fn).argtypes = [vp, i64, vp, vp, vp, vp]
    L.wl_blur_create.argtypes = [ctypes.POINTER(vp), i64, i64, dp, ci, ci, ci]
    L.wl_blur_create_gaussian.argtypes = [ctypes.POINTER(vp), i64, i64, ci, cd, ci, ci]
    L.wl_blur_destroy.argtypes = [vp]
    L.wl_blur_destroy.restype = None
    L.wl_blur_taps.argtypes = [vp, dp, ctypes.POINTER(ci)]
    L.wl_blur.argtypes = [vp, i64, vp, vp, vp]
    L.wl_blur_adjoint.argtypes = [vp, i64, vp, vp, vp]
    L.wl_blur_residual_adjoint.argtypes = [vp, i64, vp, vp, vp, vp, vp]
    L.wl_grad.argtypes = [vp, vp, i64, vp, vp, vp, vp, vp, vp]
    L.wl_fista_update.argtypes = [vp, i64, vp, vp, vp, cd, cd, cd, dp, vp]
    L.wl_grad_host.argtypes = [vp, vp, i64, vp, vp, vp, vp, vp, vp]
    L.wl_grad_adj.argtypes = [vp, vp, i64, vp, vp, vp, vp, ci, vp, vp]
    L.wl_fista_step.argtypes = [vp, vp, i64, vp, vp, vp, cd, cd, cd, vp, ci, vp, dp, vp]
    L.wl_fista_step_dev.argtypes = [vp, vp, i64, vp, vp, vp, vp, cd, cd, vp, ci, vp, vp]
    L.wl_lipschitz.argtypes = [vp, vp, ci, ctypes.c_uint64, dp, vp, vp]
    for fn in ("wl_conv_full", "wl_conv_adjoint_h", "wl_conv_adjoint_s"):
        getattr(L, fn).argtypes = [ci, i64, i64, i64, vp, vp, vp, vp]
    L.wl_bce_grad.argtypes = [ci, i64, ci, i64, i64, vp, vp, vp, ci, cd, cd, vp, vp, vp, vp]
    L.wl_last_error.restype = ctypes.c_char_p
    L.wl_launch_count.restype = ctypes.c_int64
    L.wl_version.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(status):
    if status != WL_OK:
        raise WLError(status, lib().wl_last_error().decode())


def launch_count() -> int:
    return int(lib().wl_launch_count())


def _torch():
    import torch
    return torch


def _dtype_code(dtype):
    torch = _torch()
    if dtype in (torch.float32, "float32", "f32", np.float32):
        return 0
    if dtype in (torch.float64, "float64", "f64", np.float64):
        return 1
    raise ValueError(f"unsupported dtype {dtype}")


def _stream_ptr(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _require(t, name, dtype, shape=None):
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.dtype != dtype:
        raise TypeError(f"{name} has dtype {t.dtype}, plan expects {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape[-len(shape):]) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected [..., {', '.join(map(str, shape))}]")


def _lead(t, trailing):
    """Product of the leading (batch) dims of a [..., trailing dims] tensor."""
    return int(np.prod(t.shape[:-trailing])) if t.dim() > trailing else 1


def _same_batch(B, *items):
    """Every (tensor, name, trailing) item must carry the batch B (the C side reads batch * size)."""
    for t, name, trailing in items:
        if t is not None and _lead(t, trailing) != B:
            raise ValueError(f"{name} has batch {_lead(t, trailing)} (shape {tuple(t.shape)}), expected {B}")


def _check_f(f, B):
    """f: optional float64 CUDA tensor of exactly B elements (one objective value per image)."""
    if f is not None:
        _require(f, "f", _torch().float64)
        if f.numel() != B:
            raise ValueError(f"f has {f.numel()} elements, expected one per image ({B})")


def _adopt(stream, *tensors):
    """Tensors allocated here on the current stream but used by kernels on `stream`: tell the
    caching allocator (record_stream) so their blocks are not reused while those kernels run."""
    if stream is None:
        return
    torch = _torch()
    if stream == torch.cuda.current_stream():
        return
    for t in tensors:
        if t is not None:
            t.record_stream(stream)


@dataclass(frozen=True)
class Band:
    name: str
    level: int
    offset: int
    rows: int
    cols: int
    pitch: int


class Plan:
    """Multi-level 2-D wavelet plan: W, W*, W-dagger on [h, w] images (wl_plan_create)."""

    def __init__(self, h, w, levels, filt="cdf97", bc="symmetric", dtype="float32"):
        L = lib()
        self.h, self.w, self.levels = int(h), int(w), int(levels)
        self.filter, self.bc = filt, bc
        self._dcode = _dtype_code(dtype)
        self._h = ctypes.c_void_p()
        _check(L.wl_plan_create(ctypes.byref(self._h), self.h, self.w, self.levels, FILTERS[filt], BCS[bc],
                                self._dcode))
        info = _PlanInfo()
        _check(L.wl_plan_query(self._h, ctypes.byref(info)))
        self.L = info.filter_length
        self.p_valid = int(info.p_valid)
        self.p_alloc = int(info.p_alloc)
        self.chain_h = [int(info.h[j]) for j in range(self.levels + 1)]
        self.chain_w = [int(info.w[j]) for j in range(self.levels + 1)]
        bands = [Band("LL", self.levels, *(int(v) for v in (info.band[0].offset, info.band[0].rows,
                                                            info.band[0].cols, info.band[0].pitch)))]
        i = 1
        for j in range(self.levels, 0, -1):
            for nm in ("LH", "HL", "HH"):
                b = info.band[i]
                bands.append(Band(nm, j, int(b.offset), int(b.rows), int(b.cols), int(b.pitch)))
                i += 1
        self.bands = bands

    @property
    def torch_dtype(self):
        torch = _torch()
        return torch.float64 if self._dcode == 1 else torch.float32

    def filters(self):
        """fp64 (a_lo, a_hi, d_lo, d_hi) as built by the library (host copies)."""
        arrs = [np.zeros(self.L) for _ in range(4)]
        ptrs = [a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for a in arrs]
        _check(lib().wl_plan_filters(self._h, *ptrs))
        return tuple(arrs)

    def workspace_bytes(self, op, batch, blur=None):
        return int(lib().wl_workspace_bytes(self._h, blur._h if blur is not None else None, op, int(batch)))

    def _ws(self, op, batch, blur=None, ws=None, stream=None):
        n = self.workspace_bytes(op, batch, blur)
        if ws is not None:
            if ws.numel() * ws.element_size() < n:
                raise ValueError(f"workspace too small: need {n} bytes")
            return ws
        if n == 0:
            return None
        torch = _torch()
        w = torch.empty(n, dtype=torch.uint8, device="cuda")
        _adopt(stream, w)   # the kernels on `stream` own it until they finish
        return w

    def _batch_of(self, t, trailing):
        return int(np.prod(t.shape[:-trailing])) if t.dim() > trailing else 1

    def _synthesis(self, fn, op, x, out, ws, stream):
        torch = _torch()
        _require(x, "x", self.torch_dtype, (self.p_alloc,))
        B = self._batch_of(x, 1)
        if out is None:
            out = torch.empty(x.shape[:-1] + (self.h, self.w), dtype=x.dtype, device=x.device)
            _adopt(stream, out)
        _require(out, "img", self.torch_dtype, (self.h, self.w))
        _same_batch(B, (out, "img", 2))
        ws = self._ws(op, B, ws=ws, stream=stream)
        _check(fn(self._h, B, _ptr(x), _ptr(out), _ptr(ws), _stream_ptr(stream)))
        return out

    def synthesize(self, x, out=None, ws=None, stream=None):
        """W: x [..., p_alloc] -> image [..., h, w]."""
        return self._synthesis(lib().wl_synthesize, OP_SYNTHESIZE, x, out, ws, stream)

    def analyze_adjoint(self, x, out=None, ws=None, stream=None):
        """(W-dagger)*: x [..., p_alloc] -> image [..., h, w], the transpose of analyze()."""
        return self._synthesis(lib().wl_analyze_adjoint, OP_ANALYZE_ADJOINT, x, out, ws, stream)

    def _analysis(self, fn, op, img, out, ws, stream):
        torch = _torch()
        _require(img, "img", self.torch_dtype, (self.h, self.w))
        B = self._batch_of(img, 2)
        if out is None:
            out = torch.empty(img.shape[:-2] + (self.p_alloc,), dtype=img.dtype, device=img.device)
            _adopt(stream, out)
        _require(out, "x", self.torch_dtype, (self.p_alloc,))
        _same_batch(B, (out, "x", 1))
        ws = self._ws(op, B, ws=ws, stream=stream)
        _check(fn(self._h, B, _ptr(img), _ptr(out), _ptr(ws), _stream_ptr(stream)))
        return out

    def adjoint(self, img, out=None, ws=None, stream=None):
        """W* (true adjoint of W): image [..., h, w] -> x [..., p_alloc]."""
        return self._analysis(lib().wl_adjoint, OP_ADJOINT, img, out, ws, stream)

    def analyze(self, img, out=None, ws=None, stream=None):
        """W-dagger (analysis): image [..., h, w] -> x [..., p_alloc]."""
        return self._analysis(lib().wl_analyze, OP_ANALYZE, img, out, ws, stream)

    # ---- layout helpers (pure index bookkeeping, no arithmetic) ----
    def to_packed(self, x):
        """[..., p_alloc] pitched -> [..., p_valid] packed (LL_J, (LH, HL, HH)_J..1), numpy or torch."""
        parts = []
        for b in self.bands:
            seg = x[..., b.offset:b.offset + b.rows * b.pitch].reshape(x.shape[:-1] + (b.rows, b.pitch))
            parts.append(seg[..., :b.cols].reshape(x.shape[:-1] + (b.rows * b.cols,)))
        if isinstance(x, np.ndarray):
            return np.concatenate(parts, axis=-1)
        return _torch().cat(parts, dim=-1)

    def from_packed(self, xp):
        """[..., p_valid] packed -> [..., p_alloc] pitched (padding = 0), numpy or torch."""
        if isinstance(xp, np.ndarray):
            out = np.zeros(xp.shape[:-1] + (self.p_alloc,), dtype=xp.dtype)
        else:
            out = _torch().zeros(xp.shape[:-1] + (self.p_alloc,), dtype=xp.dtype, device=xp.device)
        src = 0
        for b in self.bands:
            n = b.rows * b.cols
            dst = out[..., b.offset:b.offset + b.rows * b.pitch].reshape(out.shape[:-1] + (b.rows, b.pitch))
            dst[..., :b.cols] = xp[..., src:src + n].reshape(xp.shape[:-1] + (b.rows, b.cols))
            src += n
        return out

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib is not None:
                _lib.wl_plan_destroy(self._h)
                self._h = None
        except Exception:
            pass


class Blur:
    """Separable PSF blur R (and R*) under half-point symmetric BC (wl_blur_create*)."""

    def __init__(self, h, w, ntaps=15, sigma=3.0, taps=None, dtype="float32"):
        L = lib()
        self.h, self.w = int(h), int(w)
        self._dcode = _dtype_code(dtype)
        self._h = ctypes.c_void_p()
        if taps is None:
            _check(L.wl_blur_create_gaussian(ctypes.byref(self._h), self.h, self.w, int(ntaps), float(sigma),
                                             BCS["symmetric"], self._dcode))
        else:
            t = np.ascontiguousarray(taps, dtype=np.float64)
            _check(L.wl_blur_create(ctypes.byref(self._h), self.h, self.w,
                                    t.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), t.size, BCS["symmetric"],
                                    self._dcode))

    @property
    def torch_dtype(self):
        torch = _torch()
        return torch.float64 if self._dcode == 1 else torch.float32

    def taps(self):
        n = ctypes.c_int()
        _check(lib().wl_blur_taps(self._h, None, ctypes.byref(n)))
        arr = np.zeros(n.value)
        _check(lib().wl_blur_taps(self._h, arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(n)))
        return arr

    def _run(self, fn, img, out, stream):
        torch = _torch()
        _require(img, "in", self.torch_dtype, (self.h, self.w))
        B = int(np.prod(img.shape[:-2])) if img.dim() > 2 else 1
        if out is None:
            out = torch.empty_like(img)
            _adopt(stream, out)
        _require(out, "out", self.torch_dtype, (self.h, self.w))
        _same_batch(B, (out, "out", 2))
        _check(fn(self._h, B, _ptr(img), _ptr(out), _stream_ptr(stream)))
        return out

    def apply(self, img, out=None, stream=None):
        """R."""
        return self._run(lib().wl_blur, img, out, stream)

    def adjoint(self, img, out=None, stream=None):
        """R*."""
        return self._run(lib().wl_blur_adjoint, img, out, stream)

    def residual_adjoint(self, u, b, out=None, f=None, stream=None):
        """s = R*(R u - b); f (optional float64 [batch] CUDA tensor) <- 1/2 ||R u - b||^2."""
        torch = _torch()
        _require(u, "u", self.torch_dtype, (self.h, self.w))
        _require(b, "b", self.torch_dtype, (self.h, self.w))
        B = int(np.prod(u.shape[:-2])) if u.dim() > 2 else 1
        if out is None:
            out = torch.empty_like(u)
            _adopt(stream, out)
        _require(out, "out", self.torch_dtype, (self.h, self.w))
        _same_batch(B, (b, "b", 2), (out, "out", 2))
        _check_f(f, B)
        _check(lib().wl_blur_residual_adjoint(self._h, B, _ptr(u), _ptr(b), _ptr(out), _ptr(f),
                                              _stream_ptr(stream)))
        return out

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib is not None:
                _lib.wl_blur_destroy(self._h)
                self._h = None
        except Exception:
            pass


def grad_host(plan: Plan, blur: Blur, x, b, out=None, f=None, ws=None, stream=None):
    """wl_grad on HOST tensors (pin them for asynchronous copies): x [B, p_alloc], b [B, h, w] (CPU)
    -> g [B, p_alloc] (CPU), f (optional CPU float64 [B]).  The images are pipelined through two
    device slots (copy-in of image i+1 and copy-out of image i-1 overlap the gradient of image i);
    returns when the results are on the host."""
    torch = _torch()
    for name, t, shape in (("x", x, (plan.p_alloc,)), ("b", b, (plan.h, plan.w))):
        if not isinstance(t, torch.Tensor) or t.is_cuda or not t.is_contiguous() or t.dtype != plan.torch_dtype:
            raise ValueError(f"{name} must be a contiguous CPU tensor of {plan.torch_dtype}")
        if tuple(t.shape[-len(shape):]) != shape:
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected [..., {', '.join(map(str, shape))}]")
    B = int(np.prod(x.shape[:-1])) if x.dim() > 1 else 1
    if (int(np.prod(b.shape[:-2])) if b.dim() > 2 else 1) != B:
        raise ValueError("x and b must have the same batch")
    if out is None:
        out = torch.empty(x.shape, dtype=x.dtype, pin_memory=x.is_pinned())
    if out.is_cuda or not out.is_contiguous() or out.shape != x.shape or out.dtype != x.dtype:
        raise ValueError("out must be a contiguous CPU tensor shaped like x")
    if f is not None and (f.is_cuda or f.dtype != torch.float64 or f.numel() != B or not f.is_contiguous()):
        raise ValueError("f must be a CPU float64 tensor of batch elements")
    ws = plan._ws(OP_GRAD_HOST, B, blur=blur, ws=ws)
    st = _stream_ptr(stream)
    _check(lib().wl_grad_host(plan._h, blur._h, B, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                              ctypes.c_void_p(out.data_ptr()),
                              None if f is None else ctypes.c_void_p(f.data_ptr()), _ptr(ws), st))
    (stream or torch.cuda.current_stream()).synchronize()
    return out


ADJOINTS = {"true": 0, "pinv": 1}  # wl_adj: close the gradient with W* or with W-dagger


def grad(plan: Plan, blur: Blur, x, b, out=None, f=None, ws=None, stream=None, adjoint="true"):
    """grad f(x) = W* R* (R W x - b); f (optional float64 [batch]) <- 1/2 ||R W x - b||^2.
    adjoint="pinv" closes it with W-dagger instead of W* (the approximation P:113-117 compares)."""
    torch = _torch()
    _require(x, "x", plan.torch_dtype, (plan.p_alloc,))
    _require(b, "b", plan.torch_dtype, (plan.h, plan.w))
    B = int(np.prod(x.shape[:-1])) if x.dim() > 1 else 1
    if out is None:
        out = torch.empty_like(x)
        _adopt(stream, out)
    _require(out, "g", plan.torch_dtype, (plan.p_alloc,))
    _same_batch(B, (b, "b", 2), (out, "g", 1))
    _check_f(f, B)
    ws = plan._ws(OP_GRAD, B, blur=blur, ws=ws, stream=stream)
    if adjoint == "true":
        _check(lib().wl_grad(plan._h, blur._h, B, _ptr(x), _ptr(b), _ptr(out), _ptr(f), _ptr(ws),
                             _stream_ptr(stream)))
    else:
        _check(lib().wl_grad_adj(plan._h, blur._h, B, _ptr(x), _ptr(b), _ptr(out), _ptr(f), ADJOINTS[adjoint],
                                 _ptr(ws), _stream_ptr(stream)))
    return out


class Graph:
    """A CUDA graph of a fixed sequence of libwl calls on fixed buffers (captured once with
    torch.cuda.graph; every call is stream-ordered and allocation-free, so it is capturable).
    replay() re-runs every kernel with the captured arguments: the launch sequence of one
    wl_grad (11 kernels at cfg5) then costs one graph launch instead of 11 host launches."""

    def __init__(self, fn, warmup: int = 1):
        torch = _torch()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        n0 = launch_count()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            fn()
        self.launches = launch_count() - n0  # libwl kernels per replay

    def replay(self):
        self.graph.replay()


# ------------------------------------------------------------------ FISTA
def lipschitz(plan: Plan, blur: Blur, iters: int = 50, seed: int = 1, ws=None, stream=None) -> float:
    """lambda_max(W* R* R W) by power iteration on the GPU (wl_lipschitz; blocking)."""
    ws = plan._ws(OP_LIPSCHITZ, 1, blur=blur, ws=ws)
    out = ctypes.c_double()
    _check(lib().wl_lipschitz(plan._h, blur._h, int(iters), ctypes.c_uint64(seed), ctypes.byref(out), _ptr(ws),
                              _stream_ptr(stream)))
    return out.value


def fista_update(plan: Plan, g, x, y, t: float, lam: float, lip: float, stream=None):
    """In place: x <- soft(y - g/lip, lam/lip), y <- x + ((t-1)/t+)(x - x_old); returns t+."""
    for name, a in (("g", g), ("x", x), ("y", y)):
        _require(a, name, plan.torch_dtype, (plan.p_alloc,))
    B = plan._batch_of(x, 1)
    _same_batch(B, (g, "g", 1), (y, "y", 1))
    t_next = ctypes.c_double()
    _check(lib().wl_fista_update(plan._h, B, _ptr(g), _ptr(x), _ptr(y), float(t), float(lam), float(lip),
                                 ctypes.byref(t_next), _stream_ptr(stream)))
    return t_next.value


def fista_step(plan: Plan, blur: Blur, b, x, y, t, lam: float, lip: float, f=None, ws=None, stream=None,
               adjoint="true"):
    """One FISTA iteration on the GPU (grad f(y) then the fused prox + momentum update).

    t is either the host scalar t_k (returns t_{k+1}) or a float64 CUDA tensor of one element
    holding t_k, advanced in place on the device (wl_fista_step_dev; returns the tensor): the
    launch sequence is then identical from one iteration to the next and graph-replayable."""
    _require(b, "b", plan.torch_dtype, (plan.h, plan.w))
    _require(x, "x", plan.torch_dtype, (plan.p_alloc,))
    _require(y, "y", plan.torch_dtype, (plan.p_alloc,))
    B = plan._batch_of(x, 1)
    _same_batch(B, (b, "b", 2), (y, "y", 1))
    _check_f(f, B)
    ws = plan._ws(OP_FISTA, B, blur=blur, ws=ws, stream=stream)
    if isinstance(t, _torch().Tensor):
        _require(t, "t", _torch().float64)
        _check(lib().wl_fista_step_dev(plan._h, blur._h, B, _ptr(b), _ptr(x), _ptr(y), _ptr(t), float(lam),
                                       float(lip), _ptr(f), ADJOINTS[adjoint], _ptr(ws), _stream_ptr(stream)))
        return t
    t_next = ctypes.c_double()
    _check(lib().wl_fista_step(plan._h, blur._h, B, _ptr(b), _ptr(x), _ptr(y), float(t), float(lam), float(lip),
                               _ptr(f), ADJOINTS[adjoint], _ptr(ws), ctypes.byref(t_next), _stream_ptr(stream)))
    return t_next.value


def fista(plan: Plan, blur: Blur, b, lam: float, iters: int, lip: float = None, x0=None, stream=None,
          adjoint="true", graph: bool = False):
    """FISTA for min_x 1/2 ||R W x - b||^2 + lam ||x||_1 (Eq. (1); P:117 runs 2500 iterations).
    graph=True keeps t on the device and replays one captured iteration (wl.Graph) iters-1 times
    after a first eager iteration.  Returns (x, y, t)."""
    torch = _torch()
    B = int(np.prod(b.shape[:-2])) if b.dim() > 2 else 1
    if lip is None:
        lip = lipschitz(plan, blur, stream=stream)
    x = torch.zeros(b.shape[:-2] + (plan.p_alloc,), dtype=b.dtype, device=b.device) if x0 is None else x0.clone()
    y = x.clone()
    t_dev = torch.ones(1, dtype=torch.float64, device=b.device)
    ws = plan._ws(OP_FISTA, B, blur=blur)
    cur = torch.cuda.current_stream()
    run = stream if stream is not None else cur
    # x, y, t_dev and ws were made on the current stream: `run` starts after them, and the caller's
    # stream resumes after the last iteration (the returned x, y are safe to use there)
    run.wait_stream(cur)
    _adopt(run, x, y, t_dev, ws)
    iters = int(iters)
    if not graph:
        t = 1.0
        for _ in range(iters):
            t = fista_step(plan, blur, b, x, y, t, lam, lip, ws=ws, stream=run, adjoint=adjoint)
        cur.wait_stream(run)
        return x, y, t
    if iters == 0:
        return x, y, 1.0
    with torch.cuda.stream(run):
        step = lambda: fista_step(plan, blur, b, x, y, t_dev, lam, lip, ws=ws, adjoint=adjoint)  # noqa: E731
        step()                                   # iteration 1, eager (warms every per-kernel cache)
        if iters > 1:
            g = Graph(step, warmup=0)
            for _ in range(iters - 1):
                g.replay()
    cur.wait_stream(run)
    return x, y, float(t_dev.item())


# ------------------------------------------------------------------ Example 2
def _dtype_of(t):
    return _dtype_code(t.dtype)


def _check_1d(t, name, n, dtype=None):
    """Metadata checks of a [..., n] signal tensor; returns the flattened batch size."""
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.shape[-1] != n:
        raise ValueError(f"{name} has last dim {t.shape[-1]}, expected {n}")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} has dtype {t.dtype}, expected {dtype}")
    return int(np.prod(t.shape[:-1])) if t.dim() > 1 else 1


def conv_full(h, s, out=None, stream=None):
    """x_est = h * s, full convolution: h [..., K], s [..., N] -> [..., K+N-1]."""
    K, N = h.shape[-1], s.shape[-1]
    B = _check_1d(h, "h", K)
    if _check_1d(s, "s", N, h.dtype) != B:
        raise ValueError("h and s must have the same batch shape")
    if out is None:
        out = _torch().empty(h.shape[:-1] + (K + N - 1,), dtype=h.dtype, device=h.device)
    if _check_1d(out, "out", K + N - 1, h.dtype) != B:
        raise ValueError("out must have the batch of h")
    _check(lib().wl_conv_full(_dtype_of(h), B, K, N, _ptr(h), _ptr(s), _ptr(out), _stream_ptr(stream)))
    return out


def conv_adjoint_h(s, r, K: int, out=None, stream=None):
    """S* r = valid cross-correlation of r with s: s [..., N], r [..., K+N-1] -> [..., K]."""
    N = s.shape[-1]
    B = _check_1d(s, "s", N)
    if _check_1d(r, "r", K + N - 1, s.dtype) != B:
        raise ValueError("s and r must have the same batch shape")
    if out is None:
        out = _torch().empty(s.shape[:-1] + (K,), dtype=s.dtype, device=s.device)
    if _check_1d(out, "out", K, s.dtype) != B:
        raise ValueError("out must have the batch of s")
    _check(lib().wl_conv_adjoint_h(_dtype_of(s), B, K, N, _ptr(s), _ptr(r), _ptr(out), _stream_ptr(stream)))
    return out


def conv_adjoint_s(h, r, N: int, out=None, stream=None):
    """H* r: h [..., K], r [..., K+N-1] -> [..., N]."""
    K = h.shape[-1]
    B = _check_1d(h, "h", K)
    if _check_1d(r, "r", K + N - 1, h.dtype) != B:
        raise ValueError("h and r must have the same batch shape")
    if out is None:
        out = _torch().empty(h.shape[:-1] + (N,), dtype=h.dtype, device=h.device)
    if _check_1d(out, "out", N, h.dtype) != B:
        raise ValueError("out must have the batch of h")
    _check(lib().wl_conv_adjoint_s(_dtype_of(h), B, K, N, _ptr(h), _ptr(r), _ptr(out), _stream_ptr(stream)))
    return out


def bce_grad(h, s, x, lam_tv: float = 0.01, delta: float = 0.1, gh=None, gs=None, f=None, stream=None):
    """Gradient of the smooth part of Eq. (6), fused on the GPU.

    h [P, C, K], s [P, N], x [P, C, K+N-1] or [C, K+N-1] (one observation shared by all P problems)
    -> (gh [P, C, K], gs [P, N]); f (optional float64 [P]) <- the smooth objective.
    """
    torch = _torch()
    if h.dim() != 3 or s.dim() != 2:
        raise ValueError("h must be [P, C, K] and s [P, N]")
    P, C, K = h.shape
    N = s.shape[-1]
    _check_1d(h, "h", K)
    if _check_1d(s, "s", N, h.dtype) != P:
        raise ValueError("s must be [P, N] with the P of h")
    _check_1d(x, "x", K + N - 1, h.dtype)
    if x.dim() == 2 and tuple(x.shape) == (C, K + N - 1):
        shared = 1
    elif x.dim() == 3 and tuple(x.shape) == (P, C, K + N - 1):
        shared = 0
    else:
        raise ValueError(f"x must be [P, C, K+N-1] or [C, K+N-1], got {tuple(x.shape)}")
    gh = torch.empty_like(h) if gh is None else gh
    gs = torch.empty_like(s) if gs is None else gs
    _check_1d(gh, "gh", K, h.dtype)
    _check_1d(gs, "gs", N, h.dtype)
    if tuple(gh.shape) != tuple(h.shape) or tuple(gs.shape) != tuple(s.shape):
        raise ValueError("gh / gs must be shaped like h / s")
    _check_f(f, P)
    _check(lib().wl_bce_grad(_dtype_of(h), P, C, K, N, _ptr(h), _ptr(s), _ptr(x), shared, float(lam_tv),
                             float(delta), _ptr(gh), _ptr(gs), _ptr(f), _stream_ptr(stream)))
    return gh, gs
