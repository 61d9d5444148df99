import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1707_02018_b200 import wl
plan = wl.Plan(2048, 2048, 5, "cdf97", "symmetric_edag", "float32")
img = torch.randn(8, 2048, 2048, device="cuda"); ox = torch.empty(8, plan.p_alloc, device="cuda")
for _ in range(2): plan.adjoint(img, out=ox)
torch.cuda.synchronize()
