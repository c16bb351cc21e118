import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2501_06910_b200 as umcg
xyz, x = umcg.gen_config(3, 512, 20250113, device="cuda")
plan = umcg.Plan.build([np.linspace(0.0, 1.0, 256) for _ in range(3)], xyz)
del xyz
b = umcg.Budget(tau=1e-4, split_rho=0.5, bound_kind=1)
ar = torch.empty(plan.compress_bound("f"), dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
for _ in range(3):
    L = plan.compress_into(x, b, ar, "f"); plan.decompress_into(ar, L, out)
torch.cuda.synchronize()
os.environ["UMCG_DEC_TRACE"] = "1"
for _ in range(2):
    plan.decompress_into(ar, L, out); torch.cuda.synchronize()
