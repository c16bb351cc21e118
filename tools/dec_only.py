"""Config-3 decompress only (for ncu launch lists of the decompress chain):
python tools/dec_only.py [reps]."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_06910_b200 as umcg  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
xyz, x = umcg.gen_config(3, 512, 20250113, device="cuda")
plan = umcg.Plan.build([np.linspace(0.0, 1.0, 256) for _ in range(3)], xyz)
del xyz
b = umcg.Budget(tau=1e-4, split_rho=0.5, bound_kind=1)
ar = torch.empty(plan.compress_bound("f"), dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
L = plan.compress_into(x, b, ar, "f")
for _ in range(reps):
    plan.decompress_into(ar, L, out)
torch.cuda.synchronize()
err = (out - x).abs().max().item()
print("max err", err)
