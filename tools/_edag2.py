import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1707_02018_b200 import wl
plan = wl.Plan(2048, 2048, 5, "cdf97", "symmetric_edag", "float32")
x = torch.randn(8, plan.p_alloc, device="cuda"); oi = torch.empty(8, 2048, 2048, device="cuda")
for _ in range(2): plan.synthesize(x, out=oi)
torch.cuda.synchronize()
