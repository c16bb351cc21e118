"""Round-2 secondary measurements on config 3 (512^3 / 256^3), CUDA-event
timed, inputs resident in HBM, median of 5 after 2 warm-ups:

* multilinear g (interp.hpp:97-132) against nearest, with the per-kernel
  profile (umcg_profile_*) of one pass;
* the escape path: one +1e300 outlier under an absolute bound (escapes in
  the grid component -- exact wavefront -- and in the residual component --
  segmented lattice) against the same absolute bound without the outlier;
  umcg_serial_fallbacks() before/after.

One JSON line per case (profiles/r02_extra.jsonl)."""
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


def case(name, plan, x, b, extra=None):
    ar = torch.empty(plan.compress_bound("f"), dtype=torch.uint8, device="cuda")
    out = torch.empty(plan.n, dtype=torch.float64, device="cuda")
    L = [0]

    def c():
        L[0] = plan.compress_into(x, b, ar, "f")

    fb0 = umcg.serial_fallbacks()
    tc = timed(c)
    td = timed(lambda: plan.decompress_into(ar, L[0], out))
    fb = umcg.serial_fallbacks() - fb0
    umcg.profile_dump()
    umcg.profile(True)
    c()
    plan.decompress_into(ar, L[0], out)
    torch.cuda.synchronize()
    umcg.profile(False)
    prof = {k: round(v[0] / max(v[1], 1), 4) for k, v in umcg.profile_dump().items()}
    r = dict(case=name, n=plan.n, compress_ms=tc, decompress_ms=td, field_gbs_compress=plan.n * 8 / tc / 1e6,
             field_gbs_decompress=plan.n * 8 / td / 1e6, archive=L[0], serial_fallbacks=fb, kernels_ms=prof)
    if extra:
        r.update(extra)
    print(json.dumps(r), flush=True)
    return out


def main():
    which = sys.argv[1:] or ["multilinear", "escape"]
    xyz, x = umcg.gen_config(3, 512, 0x250106910 + 3, device="cuda")
    axes = [np.linspace(0.0, 1.0, 256) for _ in range(3)]
    plan = umcg.Plan.build(axes, xyz, keep_coords="multilinear" in which)
    del xyz
    torch.cuda.empty_cache()
    rng = float((x.max() - x.min()).item())
    if "multilinear" in which:
        for g in (0, 1):
            case(f"config3 tau_rel 1e-4 {'multilinear' if g else 'nearest'} g", plan, x,
                 umcg.Budget(tau=1e-4, g_kind=g))
    if "escape" in which:
        tau = 1e-4 * rng
        case("config3 absolute tau 1e-4*range, no outlier", plan, x, umcg.Budget(tau=tau, bound_kind=0))
        xo = x.clone()
        xo[12345] = 1e300
        out = case("config3 absolute tau 1e-4*range, one 1e300 outlier", plan, xo,
                   umcg.Budget(tau=tau, bound_kind=0))
        del out


if __name__ == "__main__":
    main()
