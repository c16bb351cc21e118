"""Throughput of the other BASELINE configs (parity cases, not bench lines):
config 2 (graded annulus), config 4 (5 fp32 variables, one batch call),
config 5 (clustered shell; seed mode at 256^3; the 9-way error split at
256^3). CUDA-event timed, inputs
resident in HBM, median of 5 after 2 warm-ups."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_06910_b200 as umcg  # noqa: E402


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def bbox_plan(xyz, g):
    lo = xyz.min(0).values.cpu().numpy()
    hi = xyz.max(0).values.cpu().numpy()
    return umcg.Plan.build([np.linspace(lo[d], hi[d], g) for d in range(xyz.shape[1])], xyz)


def run(name, plan, x, tau, n_bytes, extra=None, rho=0.5):
    b = umcg.Budget(tau=tau, split_rho=rho)
    ar = torch.empty(plan.compress_bound("f"), dtype=torch.uint8, device="cuda")
    out = torch.empty(plan.n, dtype=torch.float64, device="cuda")
    L = [0]

    def c():
        L[0] = plan.compress_into(x, b, ar, "f")

    tc = timed(c)
    td = timed(lambda: plan.decompress_into(ar, L[0], out))
    err = (out - x.double()).abs().max().item() / (tau * (x.max() - x.min()).item())
    r = dict(config=name, tau=tau, rho=rho, n=plan.n, mode=int(plan.info.mode), compress_ms=tc, decompress_ms=td,
             compress_gbs=n_bytes / tc / 1e6, decompress_gbs=n_bytes / td / 1e6, archive=L[0],
             max_err_over_tau=err)
    if extra:
        r.update(extra)
    print(json.dumps(r))


res = []
# BENCH_CFG_ONLY=2,4,5 selects configs; BENCH_CFG_QUICK=1 times config 5 at 256^3, tau 1e-2 only (A/B runs)
ONLY = [c for c in os.environ.get("BENCH_CFG_ONLY", "2,4,5").split(",") if c]
QUICK = os.environ.get("BENCH_CFG_QUICK") == "1"
# config 2: 16.7M vertices, grids 512^2 / 1024^2 / 2048^2, tau 1e-2 / 1e-4 / 1e-6
xy, x = umcg.gen_config(2, 1 << 24, 0x250106910 + 2, device="cuda")
for g in ((512, 1024, 2048) if "2" in ONLY else ()):
    plan = bbox_plan(xy, g)
    for tau in (1e-2, 1e-4, 1e-6):
        run(f"config2 grid{g}^2", plan, x, tau, x.numel() * 8)
    del plan
del xy, x
torch.cuda.empty_cache()
# config 4: 2^25 vertices, 5 fp32 variables, grid 2048^2, tau 1e-3 / 1e-5 (one batch call)
xy, vals = umcg.gen_config(4, 5793, 0x250106910 + 4, device="cuda")  # 5793^2 ~ 2^25 vertices
plan = bbox_plan(xy, 2048)
cap = 5 * plan.compress_bound("f0")
buf = torch.empty(cap, dtype=torch.uint8, device="cuda")
out32 = torch.empty_like(vals)
for tau in ((1e-3, 1e-5) if "4" in ONLY else ()):
    b = umcg.Budget(tau=tau)
    lens = [None]

    def cb():
        lens[0] = plan.compress_batch_into(vals, b, buf)

    t = timed(cb)
    td = timed(lambda: plan.decompress_batch_into(buf, lens[0], out32))
    err = max(((out32[k].double() - vals[k].double()).abs().max() / (tau * (vals[k].max() - vals[k].min()))).item()
              for k in range(5))
    print(json.dumps(dict(config="config4 batch (5 fp32 vars, umcg_compress_batch / umcg_decompress_batch fp32)",
                          tau=tau, n=plan.n, compress_ms=t, compress_gbs=vals.numel() * 4 / t / 1e6,
                          decompress_ms=td, decompress_gbs=vals.numel() * 4 / td / 1e6,
                          archive=int(np.sum(lens[0])), max_err_over_tau_fp32_out=err)))
del plan, xy, vals
torch.cuda.empty_cache()
# config 5: 200M vertices, grids 128^3 / 256^3 (seed) / 384^3 (seed)
xyz, x = umcg.gen_config(5, 200_000_000, 0x250106910 + 5, device="cuda")
for g in (((256,) if QUICK else (128, 256, 384)) if "5" in ONLY else ()):
    plan = bbox_plan(xyz, g)
    for tau in ((1e-2,) if QUICK else (1e-2, 1e-6)):
        run(f"config5 grid{g}^3", plan, x, tau, x.numel() * 8)
    if g == 256 and not QUICK:  # the error-split sweep of the config (9 splits, tau 1e-4)
        for rho in np.round(np.arange(0.1, 0.95, 0.1), 1):
            run(f"config5 grid{g}^3 split", plan, x, 1e-4, x.numel() * 8, rho=float(rho))
    del plan
