"""Host<->device copy bandwidth alone and with both directions at once
(pinned host buffers, two streams): python tools/pcie_duplex.py [GB]."""
import sys
import time

import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
n = int(gb * 1e9) // 8
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / reps
    return n * 8 / t / 1e9


run(True, True, 1)
print(f"H2D alone {run(True, False):.1f} GB/s, D2H alone {run(False, True):.1f} GB/s, "
      f"both at once {run(True, True):.1f} GB/s per direction")
