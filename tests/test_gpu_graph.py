"""CUDA-graph replay of library calls (wl.Graph): same kernels, same results as the eager calls."""
import numpy as np
import pytest

from paper_1707_02018_b200 import inputs, wl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("filt,bc", [("cdf97", "symmetric"), ("db4", "symmetric_edag"), ("db2", "periodic")])
def test_graph_replay_equals_eager(torch, filt, bc):
    h, w, J, B = 200, 176, 3, 2
    plan = wl.Plan(h, w, J, filt, bc, "float32")
    blur = wl.Blur(h, w, 15, 3.0, dtype="float32")
    rng = np.random.default_rng(0)
    x = torch.from_numpy(plan.from_packed(rng.standard_normal((B, plan.p_valid)).astype(np.float32))).cuda()
    b = torch.from_numpy(rng.standard_normal((B, h, w)).astype(np.float32)).cuda()
    g_eager = wl.grad(plan, blur, x, b)
    g = torch.empty_like(x)
    f = torch.zeros(B, dtype=torch.float64, device="cuda")
    ws = plan._ws(wl.OP_GRAD, B, blur=blur)
    graph = wl.Graph(lambda: wl.grad(plan, blur, x, b, out=g, f=f, ws=ws))
    assert graph.launches > 0
    g.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(g, g_eager)
    x.mul_(2.0)                     # replay reads the buffers' current contents
    graph.replay()
    torch.cuda.synchronize()
    assert torch.allclose(g, wl.grad(plan, blur, x, b), rtol=0, atol=0)


@pytest.mark.parametrize("B", [1, 2, 5])
def test_grad_host_pipeline_equals_device(torch, B):
    """wl_grad_host (host buffers, two pipelined device slots) = wl_grad on device copies."""
    h, w, J = 96, 80, 3
    plan = wl.Plan(h, w, J, "cdf97", "symmetric", "float32")
    blur = wl.Blur(h, w, 15, 3.0, dtype="float32")
    rng = np.random.default_rng(B)
    xh = torch.from_numpy(plan.from_packed(rng.standard_normal((B, plan.p_valid)).astype(np.float32))).pin_memory()
    bh = torch.from_numpy(rng.standard_normal((B, h, w)).astype(np.float32)).pin_memory()
    fh = torch.zeros(B, dtype=torch.float64)
    gh = wl.grad_host(plan, blur, xh, bh, f=fh)
    f = torch.zeros(B, dtype=torch.float64, device="cuda")
    g = wl.grad(plan, blur, xh.cuda(), bh.cuda(), f=f)
    assert torch.equal(gh, g.cpu())
    assert torch.allclose(fh, f.cpu(), rtol=1e-12, atol=0)
    gp = wl.grad_host(plan, blur, xh.clone(), bh.clone())   # pageable buffers: same results
    assert torch.equal(gp, gh)
