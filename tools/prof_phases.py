"""Per-kernel device times (umcg_profile events) of compress + decompress on
config 3 at a given tau: python tools/prof_phases.py [lattice] [tau ...]."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_06910_b200 as umcg  # noqa: E402

lattice = int(sys.argv[1]) if len(sys.argv) > 1 else 512
args = sys.argv[2:]
g_kind = 1 if "--multilinear" in args else 0
taus = [float(t) for t in args if not t.startswith("--")] or [1e-4]
xyz, x = umcg.gen_config(3, lattice, 20250113, device="cuda")
plan = umcg.Plan.build([np.linspace(0.0, 1.0, lattice // 2) for _ in range(3)], xyz, keep_coords=bool(g_kind))
del xyz
out = torch.empty_like(x)
for tau in taus:
    b = umcg.Budget(tau=tau, g_kind=g_kind)
    ar = torch.empty(int(plan.compress_bound("f")), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        L = plan.compress_into(x, b, ar, "f")
        plan.decompress_into(ar, L, out)
    torch.cuda.synchronize()
    umcg.profile_dump()
    umcg.profile(True)
    t0 = time.perf_counter()
    L = plan.compress_into(x, b, ar, "f")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    plan.decompress_into(ar, L, out)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    umcg.profile(False)
    d = umcg.profile_dump()
    print(f"g_kind={g_kind} tau={tau:g} archive={L} B  compress wall {1e3*(t1-t0):.3f} ms  decompress wall {1e3*(t2-t1):.3f} ms")
    for k, v in sorted(d.items(), key=lambda kv: -kv[1][0]):
        print(f"   {k:18s} {v[0]:8.3f} ms  x{v[1]}")
