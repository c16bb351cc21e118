"""Full-size parity on the BASELINE configs: the GPU path against the
unmodified reference (oracle/_ref; umc::compress / umc::decompress,
pipeline.hpp:117-148, 180-210) at the sizes BASELINE.json names.

Per case: archive bytes equal to the reference's up to codes in the
quantizer's rounding window (helpers.check_archive), the GPU decode within
1e-12 x max(range, max|x|) of the reference decode of the same archive (both
archives), the bound on every vertex for the GPU decode, and the reference's
decode of the GPU archive within the bound up to the window (a window code
differs by one bin step from the reference's, so the reference's drifted
reconstruction can exceed tau' by that window: |frac - 1/2| < 1e-6 bins).

The reference calls are single-threaded; independent ones run concurrently
on the host cores. Measured mismatch counts and drifts are appended as JSON
lines to $UMCG_PARITY_LOG when it is set (profiles/r02_fullsize_parity.jsonl).
"""
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2501_06910_b200 as umcg
from helpers import check_archive, check_decode
from oracle.bindings import Setup

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

POOL = ThreadPoolExecutor(max_workers=max(2, min(16, os.cpu_count() or 2)))


def _log(rec):
    path = os.environ.get("UMCG_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
    print(json.dumps(rec))


def _setup(plan, coords=None):
    mode, axes, assign, visited = plan.export()
    return Setup(dim=len(axes), axes=axes, mode=mode, assignments=assign, visited=visited, coords=coords)


def _bbox_axes(xyz, g):
    lo = xyz.min(0).values.cpu().numpy()
    hi = xyz.max(0).values.cpu().numpy()
    return [np.linspace(lo[d], hi[d], g) for d in range(xyz.shape[1])]


def _run_cases(plan, s, ref, oracle, fields, label, rho=0.5):
    """fields: list of (x_host f64, x_dev, tau). Reference compress and both
    reference decodes of every case run concurrently; GPU work is serial."""
    ctx = ref.ctx(s)
    want = [POOL.submit(ref.compress, s, xh, "c", tau, rho, 1, 0, 1.0, 0, 0, 0, ctx) for xh, _, tau in fields]
    got, outs = [], []
    for xh, xd, tau in fields:
        b = umcg.Budget(tau=tau, split_rho=rho, bound_kind=1)
        fb0 = umcg.serial_fallbacks()
        a = plan.compress(xd, b, name="c")
        got.append(a)
        outs.append(plan.decompress(a).cpu().numpy())
        assert umcg.serial_fallbacks() == fb0, label
    want = [w.result() for w in want]
    dec_ref_of_got = [POOL.submit(ref.decompress, s, g, ctx) for g in got]
    dec_ref_of_want = [POOL.submit(ref.decompress, s, w, ctx) for w in want]
    for k, (xh, xd, tau) in enumerate(fields):
        lab = f"{label} tau={tau}"
        mism = check_archive(got[k], want[k], s, xh, dict(tau=tau, rho=rho), oracle, lab)
        tau_abs = tau * np.ptp(xh)
        rg = dec_ref_of_got[k].result()
        drift_own, err_own = check_decode(outs[k], rg, xh, tau_abs, lab + " own archive")
        out_w = plan.decompress(want[k]).cpu().numpy()
        drift_ref, err_w = check_decode(out_w, dec_ref_of_want[k].result(), xh, tau_abs, lab + " ref archive")
        ref_err_own = float(np.max(np.abs(rg - xh))) / tau_abs
        assert ref_err_own <= 1.0 + 2e-6, (lab, ref_err_own)
        _log(dict(case=lab, n=int(xh.size), archive_bytes=len(got[k]), identical=got[k] == want[k],
                  code_mismatch=mism, drift_rel_own=drift_own, drift_rel_ref=drift_ref,
                  max_err_over_tau_gpu=err_own, max_err_over_tau_ref_decode_of_gpu=ref_err_own))
        del out_w, rg


@pytest.mark.parametrize("tau", [1e-4, 1e-2])
def test_config3_full_size_matches_reference(cuda, ref, oracle, tau):
    """Headline config 3: 512^3 = 134,217,728 vertices, grid 256^3 (uniform
    axes over the exact bbox, the GPU grid_coarsen = the reference's)."""
    import torch
    xyz, x = umcg.gen_config(3, 512, 0x250106910 + 3, device="cuda")
    plan = umcg.Plan.build([np.linspace(0.0, 1.0, 256) for _ in range(3)], xyz)
    del xyz
    torch.cuda.empty_cache()
    s = _setup(plan)
    assert s.mode == 0 and list(s.shape) == [256, 256, 256]
    _run_cases(plan, s, ref, oracle, [(x.cpu().numpy(), x, tau)], "config3 512^3/256^3")


def test_config1_spec_matches_reference(cuda, ref, oracle):
    """Config 1 at its spec: 1024^2 lattice, grid 256^2, tau 1e-3."""
    xy, x = umcg.gen_config(1, 1024, 0x250106910 + 1, device="cuda")
    plan = umcg.Plan.build([np.linspace(0.0, 1.0, 256) for _ in range(2)], xy)
    s = _setup(plan)
    _run_cases(plan, s, ref, oracle, [(x.cpu().numpy(), x, 1e-3)], "config1 1024^2/256^2")


@pytest.mark.parametrize("g", [512, 1024, 2048])
def test_config2_full_size_matches_reference(cuda, ref, oracle, g):
    """Config 2: 16,777,216 annulus vertices; grid 512^2 / 1024^2 / 2048^2
    (2048^2 is the borderline dense/seed case); the three
    bounds 1e-2 / 1e-4 / 1e-6."""
    xy, x = umcg.gen_config(2, 1 << 24, 0x250106910 + 2, device="cuda")
    plan = umcg.Plan.build(_bbox_axes(xy, g), xy)
    del xy
    s = _setup(plan)
    xh = x.cpu().numpy()
    _run_cases(plan, s, ref, oracle, [(xh, x, t) for t in (1e-2, 1e-4, 1e-6)],
               f"config2 16M/{g}^2 mode={'seed' if s.mode else 'dense'}")


def test_config4_full_size_matches_reference(cuda, ref, oracle):
    """Config 4: 2^25 vertices, five fp32 variables in one batched call per
    bound, grid 2048^2; each archive against a reference call on the widened
    values (the reference API is fp64)."""
    xy, vals = umcg.gen_config(4, 5793, 0x250106910 + 4, device="cuda")  # 5793^2 ~ 2^25
    plan = umcg.Plan.build(_bbox_axes(xy, 2048), xy)
    del xy
    s = _setup(plan)
    ctx = ref.ctx(s)
    for tau in (1e-3, 1e-5):
        archives = plan.compress_batch(vals, umcg.Budget(tau=tau), names=[f"v{k}" for k in range(5)])
        xs = [vals[k].double().cpu().numpy() for k in range(5)]
        want = [POOL.submit(ref.compress, s, xs[k], f"v{k}", tau, 0.5, 1, 0, 1.0, 0, 0, 0, ctx) for k in range(5)]
        dec = [POOL.submit(ref.decompress, s, archives[k], ctx) for k in range(5)]
        for k in range(5):
            lab = f"config4 33.5M/2048^2 var{k} tau={tau}"
            mism = check_archive(archives[k], want[k].result(), s, xs[k], dict(tau=tau), oracle, lab)
            out = plan.decompress(archives[k]).cpu().numpy()
            drift, err = check_decode(out, dec[k].result(), xs[k], tau * np.ptp(xs[k]), lab)
            _log(dict(case=lab, n=int(xs[k].size), archive_bytes=len(archives[k]),
                      identical=archives[k] == want[k].result(), code_mismatch=mism, drift_rel_own=drift,
                      max_err_over_tau_gpu=err))


@pytest.mark.parametrize("g,tau,rho", [(128, 1e-2, 0.1), (256, 1e-4, 0.5), (384, 1e-6, 0.9)])
def test_config5_full_size_matches_reference(cuda, ref, oracle, g, tau, rho):
    """Config 5: 200M clustered-shell vertices, one cell per grid of the
    sweep (128^3 dense, 256^3 and 384^3 seed mode), spanning the
    bound and error-split range."""
    import torch
    xyz, x = umcg.gen_config(5, 200_000_000, 0x250106910 + 5, device="cuda")
    plan = umcg.Plan.build(_bbox_axes(xyz, g), xyz)
    del xyz
    torch.cuda.empty_cache()
    s = _setup(plan)
    assert s.mode == (0 if g == 128 else 1)
    _run_cases(plan, s, ref, oracle, [(x.cpu().numpy(), x, tau)],
               f"config5 200M/{g}^3 mode={'seed' if s.mode else 'dense'} rho={rho}", rho=rho)


@pytest.mark.parametrize("fill", [0, 1])
def test_multilinear_verbatim_pins_g_bit_for_bit(cuda, ref, oracle, fill):
    """Multilinear g at >= 10^7 vertices (config 3, 224^3 = 11.2M vertices,
    grid 112^3) with the verbatim codec (codec 1: the raw fp64 residuals
    x - g are stored, codec.hpp:240-248): archive byte-identical to the
    reference, i.e. g (interp.hpp:97-132) bit for bit on every vertex --
    the certified Markstein quotient, the slot-hinted cell search and the
    staged corners included. Decode: bitwise equal to the reference's."""
    import torch
    xyz, x = umcg.gen_config(3, 224, 0x250106910 + 3, device="cuda")
    plan = umcg.Plan.build([np.linspace(0.0, 1.0, 112) for _ in range(3)], xyz, keep_coords=True)
    s = _setup(plan, coords=xyz.cpu().numpy())
    del xyz
    torch.cuda.empty_cache()
    xh = x.cpu().numpy()
    b = umcg.Budget(tau=1e-4, g_kind=1, fill=fill, codec_id=1)
    got = plan.compress(x, b, name="ml")
    want = ref.compress(s, xh, name="ml", tau=1e-4, g_kind=1, fill=fill, codec_id=1)
    assert got == want
    out = plan.decompress(got).cpu().numpy()
    assert np.array_equal(out.view(np.uint64), ref.decompress(s, want).view(np.uint64))
    _log(dict(case=f"multilinear verbatim config3 224^3/112^3 fill={fill}", n=int(xh.size), identical=True,
              archive_bytes=len(got)))
