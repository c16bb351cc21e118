"""Host-call timeline of the e2e paths on config 3 (lattice 512): per-call
wall times alone and inside HostPipeline."""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_06910_b200 as umcg  # noqa: E402

lat = int(sys.argv[1]) if len(sys.argv) > 1 else 512
xyz, x = umcg.gen_config(3, lat, 20250113, device="cuda")
axes = [np.linspace(0.0, 1.0, lat // 2) for _ in range(3)]
pc = umcg.Plan.build(axes, xyz)
pc2, pd, pd2 = pc.clone(), pc.clone(), pc.clone()
del xyz
b = umcg.Budget(tau=1e-4, split_rho=0.5, bound_kind=1)
cap = pc.compress_bound("f")
xh = torch.empty(x.numel(), dtype=torch.float64, pin_memory=True)
xh.copy_(x.cpu())
yh = torch.empty_like(xh).pin_memory()
slots = [torch.empty(cap, dtype=torch.uint8, pin_memory=True).numpy() for _ in range(4)]
xa, ya = xh.numpy(), yh.numpy()
for _ in range(2):
    L = pc.compress_host(xa, b, "f", out=slots[0])
    pd.decompress_host(slots[0][:L], out=ya)
t0 = time.perf_counter(); L = pc.compress_host(xa, b, "f", out=slots[0]); t1 = time.perf_counter()
pd.decompress_host(slots[0][:L], out=ya); t2 = time.perf_counter()
print(f"alone: compress_host {1e3*(t1-t0):.1f} ms, decompress_host {1e3*(t2-t1):.1f} ms")
# both at once from two threads (independent inputs)
T = {}
def c():
    a = time.perf_counter(); pc.compress_host(xa, b, "f", out=slots[1]); T["c"] = (a, time.perf_counter())
def d():
    a = time.perf_counter(); pd.decompress_host(slots[0][:L], out=ya); T["d"] = (a, time.perf_counter())
for _ in range(2):
    th = [threading.Thread(target=c), threading.Thread(target=d)]
    s0 = time.perf_counter()
    [t.start() for t in th]; [t.join() for t in th]
    s1 = time.perf_counter()
    print(f"concurrent: total {1e3*(s1-s0):.1f} ms; compress [{1e3*(T['c'][0]-s0):.1f}, {1e3*(T['c'][1]-s0):.1f}] "
          f"decompress [{1e3*(T['d'][0]-s0):.1f}, {1e3*(T['d'][1]-s0):.1f}]")
more = int(os.environ.get("E2E_MORE", "0"))  # extra workers per direction (E2E_MORE=1: 3c/3d, 2: 4c/4d)
extra_c = [pc.clone() for _ in range(more)]
extra_d = [pc.clone() for _ in range(more)]
slots += [torch.empty(cap, dtype=torch.uint8, pin_memory=True).numpy() for _ in range(2 * more)]
combos = [([pc], [pd]), ([pc, pc2], [pd]), ([pc, pc2], [pd, pd2])]
if more:
    combos = [([pc, pc2] + extra_c, [pd, pd2] + extra_d)]
for plans, pds in combos:
    pipe = umcg.HostPipeline(plans, pds, slots)
    pipe.run([xa] * 2, b, [ya] * 2, "f")
    for kp in (4, 8, 16):
        s0 = time.perf_counter(); pipe.run([xa] * kp, b, [ya] * kp, "f"); s1 = time.perf_counter()
        print(f"pipeline {len(plans)}c/{len(pds)}d plans k={kp}: {1e3*(s1-s0)/kp:.1f} ms/step")
    pipe.close()
