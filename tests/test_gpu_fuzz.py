"""Randomised parity sweep: small random meshes and budgets through the GPU
pipeline against the unmodified reference (oracle/_ref). Each case draws the
rank, the vertex count and layout (jittered lattice in random order, or a
clustered point cloud), the grid size (dense or seed mode after
grid_coarsen), the field (smooth, noisy, offset far from zero, with
outliers), the bound kind, tau over seven decades, the error split, g
(nearest / multilinear), the fill policy and the codec. The archive must be
the reference's up to rounding-window codes, errors must be the reference's
exception kinds, both decoders must agree and the bound must hold wherever
the reference's own decode meets it."""
import os

import numpy as np
import pytest

import paper_2501_06910_b200 as umcg
from helpers import check_archive
from oracle.bindings import OracleError, Setup

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    dim = int(rng.choice([2, 3]))
    if rng.random() < 0.6:
        m = int(rng.integers(20, 120 if dim == 2 else 40))
        idx = np.stack(np.meshgrid(*[np.arange(m)] * dim, indexing="ij"), -1).reshape(-1, dim)
        xyz = (idx + rng.uniform(-0.3, 0.3, idx.shape)) / (m - 1)
    else:
        n = int(rng.integers(2000, 40000))
        centres = rng.uniform(0, 1, (5, dim))
        xyz = centres[rng.integers(0, 5, n)] + rng.normal(0, 0.05, (n, dim))
    xyz = xyz[rng.permutation(len(xyz))]
    n = len(xyz)
    kind = rng.choice(["smooth", "noise", "offset", "outliers"])
    x = np.sin(6 * xyz[:, 0]) * np.cos(4 * xyz[:, 1]) + (xyz[:, 2] if dim == 3 else 0)
    if kind == "noise":
        x = x + rng.normal(0, 0.3, n)
    elif kind == "offset":
        x = x + 1000.0
    elif kind == "outliers":
        k = rng.choice(n, max(1, n // 500), replace=False)
        x[k] = rng.choice([1e12, -1e12, 1e290], len(k))
    g = int(rng.integers(4, 40 if dim == 3 else 200))
    p = dict(tau=float(10 ** rng.uniform(-8, -1)), rho=float(rng.uniform(0.1, 0.9)),
             bound_kind=int(rng.random() < 0.7), g_kind=int(rng.random() < 0.3),
             fill=int(rng.random() < 0.3), codec_id=int(rng.random() < 0.1))
    if p["bound_kind"] == 0:
        p["tau"] *= float(np.ptp(x[np.abs(x) < 1e6]) or 1.0)
    return dim, xyz, x, g, p


# UMCG_FUZZ_BASE=N shifts every seed by N (one-off wider sweeps of the same tests)
FUZZ_BASE = int(os.environ.get("UMCG_FUZZ_BASE", "0"))


@pytest.mark.parametrize("seed", range(160))
def test_random_case_matches_reference(cuda, ref, oracle, seed):
    import torch
    dim, xyz, x, g, p = _case(seed + FUZZ_BASE)
    lo, hi = xyz.min(0), xyz.max(0)
    axes = [np.linspace(lo[d], hi[d], g) for d in range(dim)]
    plan = umcg.Plan.build(axes, torch.from_numpy(np.ascontiguousarray(xyz)).cuda(), keep_coords=True)
    mode, gaxes, assign, visited = plan.export()
    s = Setup(dim=dim, axes=gaxes, mode=mode, assignments=assign, visited=visited, coords=xyz)
    b = umcg.Budget(tau=p["tau"], split_rho=p["rho"], bound_kind=p["bound_kind"], g_kind=p["g_kind"],
                    fill=p["fill"], codec_id=p["codec_id"])
    label = f"seed {seed} dim {dim} n {len(x)} g {g} mode {mode} {p}"
    try:
        want = ref.compress(s, x, name="z", tau=p["tau"], rho=p["rho"], bound_kind=p["bound_kind"],
                            g_kind=p["g_kind"], fill=p["fill"], codec_id=p["codec_id"])
    except OracleError as e:
        with pytest.raises(umcg.UmcgError) as ei:
            plan.compress(torch.from_numpy(x).cuda(), b, name="z")
        assert ei.value.kind == e.name, (label, e.name, ei.value.kind)
        return
    got = plan.compress(torch.from_numpy(x).cuda(), b, name="z")
    if p["codec_id"] == 1:
        assert got == want, label
    else:
        check_archive(got, want, s, x, p, oracle, label)
    out = plan.decompress(got).cpu().numpy()
    rd = ref.decompress(s, got)
    # decoders within 1e-12 x max(range, max|x|) -- with
    # outliers that scale is theirs: x' = approx + x2 cancels next to them in
    # both implementations, and the grid lattice's drift is relative to it
    scale = max(float(np.ptp(x)), float(np.abs(x).max()))
    assert np.max(np.abs(out - rd)) <= 1e-12 * scale, label
    tau_abs = p["tau"] * (float(np.ptp(x)) if p["bound_kind"] == 1 else 1.0)
    ok = np.abs(rd - x) <= tau_abs
    assert np.all(np.abs(out - x)[ok] <= tau_abs), label


@pytest.mark.parametrize("seed", range(96))
def test_random_codec_matches_reference(cuda, ref, oracle, seed):
    """umc::encode / umc::decode (codec.hpp:220-441) on random shapes (1-3
    axes), predictors, bounds (including 0, lossless) and values with
    outliers, bound-miss runs and exact repeats: the payload equals the
    reference's up to rounding-window codes (the N-D wavefront and the
    lossless path are exact replicas: byte-identical), both decoders agree
    and the bound holds."""
    import torch
    from helpers import check_component, lorenzo_pred
    rng = np.random.default_rng(5000 + seed + FUZZ_BASE)
    D = int(rng.integers(1, 4))
    dims = [int(rng.integers(2, {1: 20000, 2: 200, 3: 40}[D])) for _ in range(D)]
    n = int(np.prod(dims))
    pred = int(rng.integers(0, 3))
    v = np.cumsum(rng.normal(0, 1, n)) * 10 ** rng.uniform(-3, 3)
    kind = rng.choice(["plain", "outliers", "repeats", "huge"])
    if kind == "outliers":
        v[rng.choice(n, max(1, n // 300), replace=False)] = rng.choice([1e300, -1e300, 1e15])
    elif kind == "repeats":
        v[rng.choice(n, n // 3, replace=False)] = 7.25
    elif kind == "huge":
        v = v + 1e12
    tau = 0.0 if rng.random() < 0.15 else float(10 ** rng.uniform(-10, 0))
    got = umcg.encode(torch.from_numpy(v).cuda(), predictor=pred, dims=dims, tau=tau)
    want = ref.encode(v, predictor=pred, dims=dims, tau=tau)
    label = f"seed {seed} dims {dims} pred {pred} tau {tau} {kind}"
    if tau == 0.0 or (pred == 2 and D > 1):
        assert got == want, label
    else:
        rec = ref.decode(want, n)
        p = np.zeros(n) if pred == 0 else np.concatenate([[0.0], rec[:-1]])
        check_component(got, want, v, p, oracle, label)
    out = umcg.decode(got).cpu().numpy()
    rd = ref.decode(got, n)
    if tau == 0.0:
        assert np.array_equal(out.view(np.uint64), v.view(np.uint64)), label
        return
    scale = max(float(np.ptp(v)), float(np.abs(v).max()))
    assert np.max(np.abs(out - rd)) <= 1e-12 * scale, label
    assert np.max(np.abs(out - v)) <= tau, label
