"""Quick GPU check: fixture decode must take the lattice fast path."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, torch
import paper_2501_06910_b200 as umcg
from helpers import load_cases
params, cases = load_cases()
for k, s, x, archives in cases:
    plan = umcg.Plan.from_mapping(s.dim, s.axes, s.mode, s.assignments, s.visited, coords=s.coords)
    for p, ar in zip(params, archives):
        if ar.startswith(b"ERR") or p.get("tau", 1e-3) == 0:
            continue
        f0 = umcg.serial_fallbacks()
        plan.decompress(ar)
        print(k, p, "fallbacks", umcg.serial_fallbacks() - f0)
