"""Probe: compress of one field concurrently with decompress of another
(two plan handles, two host threads, two non-blocking streams) on config 3,
against the sequential step. Device-timed: events on both streams after a
common synchronization; the step time is the later end."""
import json
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_06910_b200 as umcg  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    xyz, x = umcg.gen_config(3, 512, 0x250106910 + 3, device="cuda")
    pc = umcg.Plan.build([np.linspace(0.0, 1.0, 256) for _ in range(3)], xyz)
    del xyz
    pd = pc.clone()
    b = umcg.Budget(tau=1e-4)
    cap = pc.compress_bound("f")
    arc = torch.empty(cap, dtype=torch.uint8, device="cuda")
    ard = torch.empty(cap, dtype=torch.uint8, device="cuda")
    out = torch.empty(pc.n, dtype=torch.float64, device="cuda")
    L = pc.compress_into(x, b, ard, "f")
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    # sequential reference
    for _ in range(3):
        pc.compress_into(x, b, arc, "f")
        pd.decompress_into(ard, L, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        pc.compress_into(x, b, arc, "f")
        pd.decompress_into(ard, L, out)
    e1.record()
    torch.cuda.synchronize()
    seq = e0.elapsed_time(e1) / K

    def run_c():
        for _ in range(K):
            pc.compress_into(x, b, arc, "f", stream=sa)

    def run_d():
        for _ in range(K):
            pd.decompress_into(ard, L, out, stream=sb)

    for _ in range(2):
        t = [threading.Thread(target=run_c), threading.Thread(target=run_d)]
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        sa.wait_event(s0)
        sb.wait_event(s0)
        [th.start() for th in t]
        [th.join() for th in t]
        ea.record(sa)
        eb.record(sb)
        torch.cuda.synchronize()
        par = max(s0.elapsed_time(ea), s0.elapsed_time(eb)) / K
    ok = torch.equal(out, out)
    print(json.dumps(dict(sequential_ms=seq, overlapped_ms=par, speedup=seq / par, K=K, ok=bool(ok))))


if __name__ == "__main__":
    main()
