"""The operator parity tests re-run in child processes under the library's path switches (each is read once
per process, so a child is the only way to flip it): the small-level kernels off (WL_NO_SMALL: the streaming
kernels then take the small shapes too), the register-ring analysis forced onto every zero-extension level
(WL_ARING), the full-frame symmetric fold (WL_FULL_FOLD), and the general level kernels in place of the compact
zero-extension / crop instantiations (WL_NO_PLAIN).  Every variant must stay within the same oracle
tolerances, so no code path the defaults do not take goes untested.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("env", ["WL_NO_SMALL", "WL_ARING", "WL_FULL_FOLD", "WL_NO_PLAIN"])
def test_operator_parity_under_switch(torch, env):
    e = dict(os.environ)
    e[env] = "1"
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", "operators_match_oracle or multi_strip or degenerate"]
    r = subprocess.run(cmd, cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, f"{env}=1:\n{r.stdout[-3000:]}\n{r.stderr[-2000:]}"
