"""Launch-level look at one config-2 compress + decompress (graded annulus,
16.7M vertices, grid 1024^2): python tools/prof_config2.py [tau]."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_06910_b200 as umcg  # noqa: E402

tau = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-4
xy, x = umcg.gen_config(2, 1 << 24, 0x250106910 + 2, device="cuda")
lo = xy.min(0).values.cpu().numpy()
hi = xy.max(0).values.cpu().numpy()
plan = umcg.Plan.build([np.linspace(lo[d], hi[d], 1024) for d in range(2)], xy)
b = umcg.Budget(tau=tau)
ar = torch.empty(plan.compress_bound("f"), dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
for _ in range(3):
    L = plan.compress_into(x, b, ar, "f")
    plan.decompress_into(ar, L, out)
torch.cuda.synchronize()
umcg.profile_dump()
umcg.profile(True)
plan.decompress_into(ar, L, out)
torch.cuda.synchronize()
umcg.profile(False)
for k, v in sorted(umcg.profile_dump().items(), key=lambda kv: -kv[1][0]):
    print(f"   {k:18s} {v[0]:8.3f} ms  x{v[1]}")
