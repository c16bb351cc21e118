"""Escapes in parallel (codec.hpp:300-326 encode, 408-437 decode).

An element escapes when its quantum leaves int32 or its reconstruction misses
the bound in floating point; the reference stores (index, value) and restarts
its chain from the exact value. The GPU path handles them without the
one-thread replica: lorenzo_1d components by the segmented lattice
(escape.cu), 2-/3-D Lorenzo grids by the exact hyperplane wavefront
(codes.cu). Checked against the unmodified reference: identical escape
records, codes equal up to the rounding window, decoders within 1e-12, the
bound on every element, and umcg_serial_fallbacks() unchanged.
"""
import numpy as np
import pytest

import paper_2501_06910_b200 as umcg
from helpers import check_archive, check_component, check_decode, parse_payload
from oracle.bindings import Setup

pytestmark = pytest.mark.gpu


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float64)).cuda()


def _tol(v):
    """1e-12 relative, elementwise: to the field's normal range (outliers
    excluded) or to the element's own magnitude when larger."""
    normal = np.abs(v[np.abs(v) < 1e100])
    return 1e-12 * np.maximum(normal.max() if normal.size else 1.0, np.abs(v))


def _codec_case(ref, oracle, v, predictor, dims, tau, expect_parallel=True):
    fb0 = umcg.serial_fallbacks()
    got = umcg.encode(dev(v), predictor=predictor, dims=dims, tau=tau)
    want = ref.encode(v, predictor=predictor, dims=dims, tau=tau)
    g = parse_payload(got, oracle.rle_decompress)
    r = parse_payload(want, oracle.rle_decompress)
    assert len(r["esc"]) > 0, "the case must produce escapes"
    rec = ref.decode(want, v.size)
    if predictor == 1 or len(dims) == 1:
        pred = np.concatenate([[0.0], rec[:-1]])
        check_component(got, want, v, pred, oracle, f"pred{predictor} tau={tau}")
    else:
        assert got == want  # the wavefront is an exact replica
    out = umcg.decode(got).cpu().numpy()
    out_ref = umcg.decode(want).cpu().numpy()
    tol = _tol(v)
    assert np.all(np.abs(out - ref.decode(got, v.size)) <= tol)
    assert np.all(np.abs(out_ref - rec) <= tol)
    assert np.max(np.abs(out - v)) <= tau
    if expect_parallel:
        assert umcg.serial_fallbacks() == fb0
    return len(g["esc"])


@pytest.mark.parametrize("n_out", [1, 100, 10000])
def test_1d_outliers_segmented(cuda, ref, oracle, n_out):
    """lorenzo_1d with +-1e300 outliers (each escapes, and so does its
    successor, whose prediction is the outlier): the chain restarts from the
    successor's exact value."""
    rng = np.random.default_rng(n_out)
    n = 1 << 20
    v = np.cumsum(rng.normal(0, 1e-3, n)) + np.sin(np.arange(n) * 1e-4)
    idx = rng.choice(n, n_out, replace=False)
    v[idx] = np.where(rng.random(n_out) < 0.5, 1e300, -1e300)
    ne = _codec_case(ref, oracle, v, 1, [n], 1e-4)
    assert ne >= n_out


def test_1d_int32_overflow_escapes(cuda, ref, oracle):
    """Quanta beyond int32 from a tiny bound on a random walk with jumps.
    |v| / bin reaches 5e9 > 2^30: outside the lattice regime (the serial
    chain's drift exceeds the rounding window), so the exact replica runs --
    counted, and the archive is the reference's bit for bit."""
    rng = np.random.default_rng(5)
    n = 300000
    v = np.cumsum(rng.normal(0, 1.0, n))
    v[rng.choice(n, 500, replace=False)] += rng.normal(0, 1e4, 500)
    fb0 = umcg.serial_fallbacks()
    _codec_case(ref, oracle, v, 1, [n], 1e-7, expect_parallel=False)
    assert umcg.serial_fallbacks() > fb0
    assert umcg.encode(dev(v), predictor=1, dims=[n], tau=1e-7) == ref.encode(v, predictor=1, dims=[n], tau=1e-7)


def test_1d_bound_miss_huge_runs(cuda, ref, oracle):
    """Runs of huge, close values: reconstructions miss the bound in floating
    point (bound-miss escapes, not overflow). Outside the lattice regime the
    one-thread replica may run; the result must still be the reference's."""
    rng = np.random.default_rng(9)
    n = 50000
    v = np.sin(np.arange(n) * 1e-2)
    for s in rng.choice(n - 40, 20, replace=False):
        v[s:s + 30] = 3e12 + rng.normal(0, 1e-3, 30)
    _codec_case(ref, oracle, v, 1, [n], 1e-5, expect_parallel=False)


@pytest.mark.parametrize("dims", [[300, 200], [64, 48, 40]])
def test_nd_outliers_wavefront_exact(cuda, ref, oracle, dims):
    """2-/3-D Lorenzo with outliers: the outlier and the neighbours whose
    prediction it enters escape; byte-exact with the reference."""
    rng = np.random.default_rng(len(dims))
    n = int(np.prod(dims))
    v = np.cumsum(rng.normal(size=n)).reshape(dims) * 1e-2
    v = v.ravel()
    v[rng.choice(n, 40, replace=False)] = 1e200
    _codec_case(ref, oracle, v, 2, dims, 1e-4)


@pytest.mark.parametrize("n_out", [1, 100, 10000])
def test_pipeline_outliers_absolute_bound(cuda, ref, oracle, n_out):
    """The archive pipeline on a config-3 sample (lattice 96^3, grid 48^3)
    with +-1e300 outliers under an absolute bound: escapes in the grid
    component (cluster means, wavefront) and in the residual component
    (segmented lattice)."""
    xyz, x = umcg.gen_config(3, 96, 20250113, device="cuda")
    plan = umcg.Plan.build([np.linspace(0.0, 1.0, 48) for _ in range(3)], xyz)
    mode, gaxes, assign, visited = plan.export()
    s = Setup(dim=3, axes=gaxes, mode=mode, assignments=assign, visited=visited)
    rng = np.random.default_rng(n_out)
    xh = x.cpu().numpy()
    idx = rng.choice(xh.size, n_out, replace=False)
    xh[idx] = np.where(rng.random(n_out) < 0.5, 1e300, -1e300)
    tau = 1e-3
    fb0 = umcg.serial_fallbacks()
    got = plan.compress(dev(xh), umcg.Budget(tau=tau, bound_kind=0), name="o")
    assert umcg.serial_fallbacks() == fb0
    want = ref.compress(s, xh, name="o", tau=tau, bound_kind=0)
    p = dict(tau=tau, bound_kind=0)
    check_archive(got, want, s, xh, p, oracle, f"outliers {n_out}")
    out = plan.decompress(got).cpu().numpy()
    assert umcg.serial_fallbacks() == fb0
    rd = ref.decompress(s, got)
    tol = _tol(xh)
    assert np.all(np.abs(out - rd) <= tol)
    # x' = approx + x2' cancels catastrophically next to a 1e299 cluster mean
    # (pipeline.hpp:206-208) for the reference as well: the bound is checked
    # wherever the reference's own decode meets it
    ok = np.abs(rd - xh) <= tau
    assert ok.mean() > 0.5
    assert np.all(np.abs(out - xh)[ok] <= tau)
    out_w = plan.decompress(want).cpu().numpy()
    assert np.all(np.abs(out_w - ref.decompress(s, want)) <= tol)


@pytest.mark.parametrize("layout", ["edges", "tile_boundaries", "runs"])
def test_1d_escape_positions(cuda, ref, oracle, layout):
    """Escapes where the fixed-point scan's carries matter: the first and the
    last element, both sides of every 2048-element tile boundary and of the
    8-element thread boundaries, and runs of consecutive outliers crossing
    them (each run's second element codes q = 0 against the first: the exact
    segment after an escape)."""
    rng = np.random.default_rng(hash(layout) % 2**32)
    n = 5 * 2048 + 3
    v = np.cumsum(rng.normal(0, 1e-3, n))
    if layout == "edges":
        idx = [0, 1, n - 2, n - 1]
    elif layout == "tile_boundaries":
        idx = sorted({k + d for k in range(2048, n, 2048) for d in (-1, 0)} | {7, 8, 15, 16})
    else:
        idx = [i for k in range(2040, n, 2048) for i in range(k, min(n, k + 12))]
    v[idx] = 1e300
    _codec_case(ref, oracle, v, 1, [n], 1e-4)


def test_pipeline_outliers_seed_mode(cuda, ref, oracle):
    """Seed-mode grid (config-5 shell at 2^19 vertices, 96^3: visited fraction
    under 0.35, the grid component is lorenzo_1d over the visited nodes) with
    outliers under an absolute bound: escapes in both 1-D components
    (segmented lattice), against the reference."""
    xyz, x = umcg.gen_config(5, 1 << 19, 20250115, device="cuda")
    lo = xyz.min(0).values.cpu().numpy()
    hi = xyz.max(0).values.cpu().numpy()
    plan = umcg.Plan.build([np.linspace(lo[d], hi[d], 96) for d in range(3)], xyz)
    mode, gaxes, assign, visited = plan.export()
    assert mode == 1
    s = Setup(dim=3, axes=gaxes, mode=mode, assignments=assign, visited=visited)
    rng = np.random.default_rng(77)
    xh = x.cpu().numpy()
    idx = rng.choice(xh.size, 300, replace=False)
    xh[idx] = np.where(rng.random(300) < 0.5, 1e300, -1e300)
    tau = 1e-3
    fb0 = umcg.serial_fallbacks()
    got = plan.compress(dev(xh), umcg.Budget(tau=tau, bound_kind=0), name="s")
    assert umcg.serial_fallbacks() == fb0
    want = ref.compress(s, xh, name="s", tau=tau, bound_kind=0)
    check_archive(got, want, s, xh, dict(tau=tau, bound_kind=0), oracle, "seed outliers")
    out = plan.decompress(got).cpu().numpy()
    assert umcg.serial_fallbacks() == fb0
    rd = ref.decompress(s, got)
    assert np.all(np.abs(out - rd) <= _tol(xh))
    ok = np.abs(rd - xh) <= tau
    assert np.all(np.abs(out - xh)[ok] <= tau)
