"""Build libwl.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension machinery).

The shared library links the CUDA runtime statically and exports only the C ABI of
include/wl.h.  `build()` is called by __graft_entry__.build() and lazily by the binding.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libwl.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-I", INCLUDE,
         "--expt-relaxed-constexpr", "-diag-suppress", "177"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(INCLUDE, "*.h")))


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False, lib: str = LIB, obj: str = OBJ,
          defines=()) -> str:
    """Compile every csrc source for sm_100a and link `lib` (defines: extra -D flags for A/B builds)."""
    os.makedirs(obj, exist_ok=True)
    hdr_t = max([_mtime(h) for h in _headers()] + [_mtime(__file__)])
    objs, cmds = [], []
    for src in _sources():
        o = os.path.join(obj, os.path.basename(src) + ".o")
        objs.append(o)
        if force or _mtime(o) < max(_mtime(src), hdr_t):
            cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", o]
            if ptxas_v and src.endswith(".cu"):
                cmd += ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            cmds.append(cmd)
    changed = force or bool(cmds)
    # the translation units are independent: compile them concurrently (the template-heavy
    # kernel files dominate, one process each)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for _ in ex.map(subprocess.check_call, cmds):
            pass
    if changed or _mtime(lib) < max(_mtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib, *objs, "-lcuda"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_v="-v" in sys.argv)
    print(LIB)
