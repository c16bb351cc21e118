"""Compress phase timeline (UMCG_COMP_TRACE) on config 3: python tools/comp_trace.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_06910_b200 as umcg
xyz, x = umcg.gen_config(3, 512, 20250113, device="cuda")
plan = umcg.Plan.build([np.linspace(0.0, 1.0, 256) for _ in range(3)], xyz)
del xyz
b = umcg.Budget(tau=1e-4, split_rho=0.5, bound_kind=1)
ar = torch.empty(plan.compress_bound("f"), dtype=torch.uint8, device="cuda")
for _ in range(3):
    plan.compress_into(x, b, ar, "f")
torch.cuda.synchronize()
os.environ["UMCG_COMP_TRACE"] = "1"
for _ in range(2):
    plan.compress_into(x, b, ar, "f")
    torch.cuda.synchronize()
