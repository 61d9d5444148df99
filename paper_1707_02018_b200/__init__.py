"""B200-native hot path of arXiv 1707.02018 (Folberth & Becker): W, W*, W-dagger, R, R*, grad f.

The compute lives in libwl.so (hand-written sm_100a CUDA, C ABI in include/wl.h);
`wl` is the ctypes binding.  There is no CPU fallback.
"""
from . import wl  # noqa: F401
from .wl import Blur, Plan, WLError, grad  # noqa: F401
