import time, torch, sys, os
sys.path.insert(0, os.getcwd())
from paper_1707_02018_b200 import inputs, wl
for cfg in (5, 2):
    c = inputs.CONFIGS[cfg]
    plan = wl.Plan(c.h, c.w, c.levels, c.filt, c.bc, c.dtype); B = c.batch
    blur = wl.Blur(c.h, c.w, 15, 3.0, dtype=c.dtype)
    x = torch.randn(B, plan.p_alloc, device="cuda", dtype=plan.torch_dtype)
    img = torch.randn(B, c.h, c.w, device="cuda", dtype=plan.torch_dtype)
    g = torch.empty_like(x); ws = plan._ws(wl.OP_GRAD, B, blur=blur); wsa = plan._ws(wl.OP_ADJOINT, B)
    for _ in range(5): wl.grad(plan, blur, x, img, out=g, ws=ws)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(30): wl.grad(plan, blur, x, img, out=g, ws=ws)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(cfg, "grad host us/call", (t1 - t) / 30 * 1e6, "total us/call", (t2 - t) / 30 * 1e6)
    t = time.perf_counter()
    for _ in range(30): plan.adjoint(img, out=g, ws=wsa)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(cfg, "adjoint host us/call", (t1 - t) / 30 * 1e6, "total us/call", (t2 - t) / 30 * 1e6)
