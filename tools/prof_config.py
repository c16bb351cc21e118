"""Per-kernel device times (umcg_profile events) of one compress + decompress
of config 2/5 on a bounding-box grid: python tools/prof_config.py <config>
<vertices> <grid> [tau ...]."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_06910_b200 as umcg  # noqa: E402

# UMCG_PROF_RANGE=compress|decompress: cudaProfilerStart/Stop around that
# call (ncu --profile-from-start off) for a launch list of exactly one call
RANGE = os.environ.get("UMCG_PROF_RANGE", "")
cfg, nv, g = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
taus = [float(t) for t in sys.argv[4:]] or [1e-2]
xyz, x = umcg.gen_config(cfg, nv, 0x250106910 + cfg, device="cuda")
lo = xyz.min(0).values.cpu().numpy()
hi = xyz.max(0).values.cpu().numpy()
plan = umcg.Plan.build([np.linspace(lo[d], hi[d], g) for d in range(xyz.shape[1])], xyz)
del xyz
print(f"config {cfg} n={plan.n} grid {g} mode={int(plan.info.mode)}")
ar = torch.empty(plan.compress_bound("f"), dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
for tau in taus:
    b = umcg.Budget(tau=tau)
    for _ in range(3):
        L = plan.compress_into(x, b, ar, "f")
        plan.decompress_into(ar, L, out)
    torch.cuda.synchronize()
    for phase in ("compress", "decompress"):
        umcg.profile_dump()
        umcg.profile(True)
        t0 = time.perf_counter()
        if RANGE == phase:
            torch.cuda.profiler.start()
        if phase == "compress":
            L = plan.compress_into(x, b, ar, "f")
        else:
            plan.decompress_into(ar, L, out)
        torch.cuda.synchronize()
        if RANGE == phase:
            torch.cuda.profiler.stop()
        t1 = time.perf_counter()
        umcg.profile(False)
        d = umcg.profile_dump()
        print(f"tau={tau:g} {phase} wall {1e3 * (t1 - t0):.3f} ms archive={L}")
        for k, v in sorted(d.items(), key=lambda kv: -kv[1][0]):
            print(f"   {k:18s} {v[0]:8.3f} ms  x{v[1]}")
