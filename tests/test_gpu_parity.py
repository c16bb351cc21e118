"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracles.

Bar (BASELINE.json north_star): archives / payloads byte-identical to the
reference, except codes whose value sits in the quantizer's rounding window
(|frac((v - p_ref)/bin) - 0.5| < WINDOW, p_ref the reference's serial
prediction); decoded values within 1e-12 x max(range, max|x|) of the
reference's decode; the error bound on 100% of vertices.
"""
import os

import numpy as np
import pytest

import paper_2501_06910_b200 as umcg
from oracle.bindings import Setup
from helpers import (GOLDEN, REL_TOL, WINDOW, check_archive, check_component, check_decode, load_cases,
                     load_seed7, lorenzo_pred, parse_archive, parse_payload, window_distance)

pytestmark = pytest.mark.gpu



def plan_for(s, coords=True):
    return umcg.Plan.from_mapping(s.dim, s.axes, s.mode, s.assignments, s.visited,
                                  coords=s.coords if coords else None)


def budget_of(p):
    return umcg.Budget(tau=p.get("tau", 1e-3), split_rho=p.get("rho", 0.5),
                       bound_kind=p.get("bound_kind", 1), g_kind=p.get("g_kind", 0),
                       fill=p.get("fill", 0))


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float64)).cuda()


# ---------------------------------------------------------------------------


def test_golden_archive_bit_exact(cuda):
    s, x, ar = load_seed7()
    plan = plan_for(s)
    got = plan.compress(dev(x), umcg.Budget(tau=1e-3, split_rho=0.5, bound_kind=1), name="white-noise")
    assert got == ar
    out = plan.decompress(ar).cpu().numpy()
    assert np.max(np.abs(out - x)) <= 1e-3 * np.ptp(x)


def test_plan_digest_matches_reference(cuda, ref):
    s, x, ar = load_seed7()
    assert plan_for(s).digest == ref.mapping_digest(s) == parse_archive(ar)["digest"]


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("n", [1, 255, 16383, 16384, 16385, 50001])
def test_parallel_digest_matches_reference(cuda, ref, mode, n):
    """mapping_digest (serialize.hpp:255-267, 300-303): the device FNV-1a (chunk
    maps keyed by the low byte, digest.cu) on chunk-boundary sizes, ids with
    1-3 significant bytes and zero ids, and a seed-mode mapping (assignments
    into a visited list, the list hashed after them)."""
    rng = np.random.default_rng(1000 * mode + n)
    g = 300  # 90000 nodes: ids up to 3 bytes
    axes = [np.linspace(0.0, 1.0, g), np.linspace(0.0, 1.0, g)]
    if mode == 0:
        a = rng.integers(0, g * g, n).astype(np.uint64)
        a[rng.random(n) < 0.2] = 0
        small = rng.random(n) < 0.2
        a[small] = rng.integers(0, 256, int(small.sum())).astype(np.uint64)
        s = Setup(2, axes, 0, a)
    else:
        nv = min(n, 977)
        vis = np.sort(rng.choice(g * g, nv, replace=False)).astype(np.uint64)
        a = rng.integers(0, nv, n).astype(np.uint64)
        s = Setup(2, axes, 1, a, vis)
    assert plan_for(s, coords=False).digest == ref.mapping_digest(s)


@pytest.mark.parametrize("case_idx", range(7))
def test_fixture_cases(cuda, case_idx, ref, oracle):
    params, cases = load_cases()
    k, s, x, archives = cases[case_idx]
    plan = plan_for(s)
    dx = dev(x)
    for p, ref_ar in zip(params, archives):
        label = f"case{k} {p}"
        b = budget_of(p)
        if ref_ar.startswith(b"ERR:"):
            with pytest.raises(umcg.UmcgError) as ei:
                plan.compress(dx, b, name=f"case{k}")
            assert ei.value.kind == "seed_mode_unsupported"
            continue
        fb0 = umcg.serial_fallbacks()
        got = plan.compress(dx, b, name=f"case{k}")
        check_archive(got, ref_ar, s, x, p, oracle, label)
        tau_abs = p.get("tau", 1e-3) * (np.ptp(x) if p.get("bound_kind", 1) == 1 else 1.0)
        # GPU decode of the reference archive and of our own archive
        ref_dec = ref.decompress(s, ref_ar)
        out_ref_ar = plan.decompress(ref_ar).cpu().numpy()
        check_decode(out_ref_ar, ref_dec, x, tau_abs, label + " gpu(ref archive)")
        out_own = plan.decompress(got).cpu().numpy()
        check_decode(out_own, ref.decompress(s, got), x, tau_abs, label + " gpu(own archive)")
        if p.get("tau", 1e-3) > 0:
            # lossy data in the lattice regime never takes the one-thread exact path
            assert umcg.serial_fallbacks() == fb0, label


def test_codec_known_answers(cuda, ref):
    z = np.load(os.path.join(GOLDEN, "codec.npz"))
    assert umcg.encode(dev(z["worked_in"]), predictor=0, tau=0.05) == z["worked_payload"].tobytes()
    assert umcg.decode(z["worked_payload"].tobytes()).cpu().numpy()[0] == 0.4
    # escapes: exact serial path
    assert umcg.encode(dev(z["esc_in"]), predictor=1, tau=1e-12) == z["esc_payload"].tobytes()
    out = umcg.decode(z["esc_payload"].tobytes()).cpu().numpy()
    assert np.all(np.abs(out - z["esc_in"]) <= 1e-12)
    for pred in (0, 1):
        pl = z[f"lossless_payload{pred}"].tobytes()
        assert umcg.encode(dev(z["lossless_in"]), predictor=pred, tau=0.0) == pl
        back = umcg.decode(pl).cpu().numpy()
        assert np.array_equal(back.view(np.uint64), z["lossless_in"].view(np.uint64))
    for t in (0.0, 1e-6, 0.5):
        pl = z[f"zeros_payload_{t}"].tobytes()
        assert umcg.encode(dev(np.zeros(10000)), predictor=1, tau=t) == pl
        assert np.array_equal(umcg.decode(pl).cpu().numpy(), np.zeros(10000))
    nd = z["nd_in"]
    assert umcg.encode(dev(nd), predictor=2, dims=[17, 9, 5], tau=0.0) == z["nd0_payload"].tobytes()
    back = umcg.decode(z["nd0_payload"].tobytes()).cpu().numpy()
    assert np.array_equal(back.view(np.uint64), nd.view(np.uint64))
    got = umcg.encode(dev(nd), predictor=2, dims=[17, 9, 5], tau=1e-3)
    assert got == z["nd_payload"].tobytes()


def test_codec_random_walk_and_smooth(cuda, ref, oracle):
    z = np.load(os.path.join(GOLDEN, "codec.npz"))
    w = z["walk_in"]
    got = umcg.encode(dev(w), predictor=1, tau=1e-3)
    rp = z["walk_payload"].tobytes()
    rec = oracle.decode(rp)
    check_component(got, rp, w, np.concatenate([[0.0], rec[:-1]]), oracle, "walk")
    out = umcg.decode(got).cpu().numpy()
    assert np.max(np.abs(out - w)) <= 1e-3
    for t in (1e-6, 1e-5, 1e-4, 1e-3, 1e-2):
        pl = z[f"smooth_payload_{t}"].tobytes()
        sm = z["smooth_in"]
        got = umcg.encode(dev(sm), predictor=1, tau=t)
        rec = oracle.decode(pl)
        check_component(got, pl, sm, np.concatenate([[0.0], rec[:-1]]), oracle, f"smooth{t}")
        back = umcg.decode(pl).cpu().numpy()
        assert np.max(np.abs(back - rec)) <= REL_TOL * 10.0
        assert np.max(np.abs(back - sm)) <= t


def test_codec_bound_random_shapes(cuda, ref, oracle):
    """test_codec.cpp:74-104 'hard error bound across shapes and tolerances'."""
    rng = np.random.default_rng(100)
    for trial in range(40):
        nd = 1 + int(rng.integers(0, 3))
        dims = [1 + int(rng.integers(0, 400 if d == 0 else 20)) for d in range(nd)]
        n = int(np.prod(dims))
        v = rng.uniform(-50, 50, n)
        if trial % 3 == 0:
            v = np.cumsum(v * 0.01)
        tau = 10.0 ** (-1 - int(rng.integers(0, 6))) * np.ptp(v) if n > 1 else 1e-3
        if tau == 0:
            tau = 1e-3
        pred = 1 if nd == 1 else 2
        got = umcg.encode(dev(v), predictor=pred, dims=dims, tau=tau)
        rp = ref.encode(v, predictor=pred, dims=dims, tau=tau)
        rec = oracle.decode(rp)
        p_ref = np.concatenate([[0.0], rec[:-1]]) if nd == 1 else lorenzo_pred(rec, dims)
        check_component(got, rp, v, p_ref, oracle, f"shape{dims}")
        out = umcg.decode(got).cpu().numpy()
        assert np.all(np.abs(out - v) <= tau)
        out_r = umcg.decode(rp).cpu().numpy()
        assert np.all(np.abs(out_r - v) <= tau)


def test_gpu_grid_coarsen_matches_reference(cuda, ref):
    import torch
    rng = np.random.default_rng(5)
    for dim, m, gsz in [(2, 90, 30), (3, 20, 9), (2, 60, 200)]:
        h = 1.0 / (m - 1)
        idx = np.stack(np.meshgrid(*([np.arange(m)] * dim), indexing="ij"), -1).reshape(-1, dim)
        coords = idx * h + rng.uniform(-0.3, 0.3, idx.shape) * h * ((idx > 0) & (idx < m - 1))
        coords = coords[rng.permutation(len(coords))]
        if gsz == 200:  # sparse occupancy -> seed mode
            coords = coords[: len(coords) // 7]
        axes = [np.linspace(0, 1, gsz) for _ in range(dim)]
        s, frac = ref.grid_coarsen(dim, coords, axes)
        plan = umcg.Plan.build(axes, torch.from_numpy(coords).cuda())
        mode, gaxes, assign, visited = plan.export()
        assert mode == s.mode
        for a, b in zip(gaxes, s.axes):
            assert np.array_equal(a, b)
        assert np.array_equal(assign, s.assignments)
        if mode == 1:
            assert np.array_equal(visited, s.visited)
        assert plan.digest == ref.mapping_digest(s)
        assert plan.info.visited_fraction == frac


def test_errors_follow_reference_taxonomy(cuda, ref):
    params, cases = load_cases()
    k, s, x, archives = cases[0]
    plan = plan_for(s)
    dx = dev(x)
    ar = archives[1]
    # wrong mapping -> mapping_mismatch (pipeline.hpp:188-189)
    k2, s2, x2, _ = cases[1]
    with pytest.raises(umcg.UmcgError) as e:
        plan_for(s2).decompress(ar)
    assert e.value.kind == "mapping_mismatch"
    # truncation -> malformed_file (deserialize_archive)
    for cut in (len(ar) - 1, len(ar) // 2, 10, 3):
        with pytest.raises(umcg.UmcgError) as e:
            plan.decompress(ar[:cut])
        assert e.value.kind == "malformed_file"
    # non-finite input
    bad = x.copy()
    bad[5] = np.nan
    with pytest.raises(umcg.UmcgError) as e:
        plan.compress(dev(bad))
    assert e.value.kind == "non_finite_value"
    # budget
    for b in (umcg.Budget(split_rho=1.0), umcg.Budget(split_rho=0.0), umcg.Budget(tau=-1.0)):
        with pytest.raises(umcg.UmcgError) as e:
            plan.compress(dx, b)
        assert e.value.kind == "budget_inadmissible"
    # non-finite beats budget (validate_field runs first)
    with pytest.raises(umcg.UmcgError) as e:
        plan.compress(dev(bad), umcg.Budget(split_rho=2.0))
    assert e.value.kind == "non_finite_value"
    with pytest.raises(umcg.UmcgError) as e:
        plan.compress(dx, umcg.Budget(codec_id=17))
    assert e.value.kind == "unknown_codec"
    # corrupt payload bytes inside the residual stream -> corrupt_payload
    a = parse_archive(ar)
    p2_off = ar.index(a["p2"])
    broken = bytearray(ar)
    broken[p2_off + 37] = 0x07  # first RLE token tag -> unknown token
    with pytest.raises(umcg.UmcgError) as e:
        plan.decompress(bytes(broken))
    assert e.value.kind == "corrupt_payload"
    # truncated component payloads -> corrupt_payload (test_codec.cpp:147-157)
    z = np.load(os.path.join(GOLDEN, "codec.npz"))
    pl = z["walk_payload"].tobytes()
    for cut in (len(pl) - 1, len(pl) // 2, 10):
        with pytest.raises(umcg.UmcgError) as e:
            umcg.decode(pl[:cut], n_capacity=len(z["walk_in"]))
        assert e.value.kind == "corrupt_payload"


def test_determinism_and_host_path(cuda):
    params, cases = load_cases()
    k, s, x, archives = cases[5]
    plan = plan_for(s)
    a1 = plan.compress(dev(x), umcg.Budget(tau=1e-4))
    a2 = plan.compress(dev(x), umcg.Budget(tau=1e-4))
    a3 = plan.compress_host(x, umcg.Budget(tau=1e-4))
    assert a1 == a2 == a3
    y = plan.decompress_host(a1)
    assert np.array_equal(y, plan.decompress(a1).cpu().numpy())


@pytest.mark.parametrize("seed", range(6))
def test_rle_stream_patterns_bit_exact(cuda, ref, seed):
    """Zero-run structure at every scale (runs of 0..40 zero codes, all-zero
    tiles, runs crossing the 2048-code tiles, long literals) through the
    predictor=none path, whose codes are exact, so payloads must match the
    reference byte for byte (lossless.hpp:24-51 token structure)."""
    rng = np.random.default_rng(1000 + seed)
    n = [5000, 70000, 300000, 2048 * 3, 2048 * 5 + 7, 1][seed % 6] if seed < 6 else 10000
    q = np.zeros(n, np.int64)
    i = 0
    while i < n:
        if rng.random() < 0.5:
            run = int(rng.choice([1, 3, 7, 8, 9, 15, 40, 2048, 5000]))
            i += run  # zeros
        else:
            lit = int(rng.integers(1, 60))
            q[i:i + lit] = rng.integers(-300, 300, size=min(lit, n - i))
            i += lit
    if seed == 4:
        q[:] = 0
        q[-1] = 5  # one long run then a literal
    tau = 0.5
    v = q.astype(np.float64) * (2 * tau)
    got = umcg.encode(dev(v), predictor=0, tau=tau)
    want = ref.encode(v, predictor=0, tau=tau)
    assert got == want
    back = umcg.decode(want).cpu().numpy()
    assert np.array_equal(back, ref.decode(want, n))


def _token_dense_codes(rng, n, long_lits=False):
    """Codes whose zero-RLE stream is dense with tokens (short literals between
    8..12-zero runs), optionally interleaved with literals spanning many
    8 KiB parse chunks."""
    q = np.zeros(n, np.int64)
    i = 0
    while i < n:
        if long_lits and rng.random() < 0.002:
            lit = int(rng.integers(20000, 120000))
            q[i:i + lit] = rng.integers(-3, 4, size=min(lit, n - i)) | 1
            i += lit
        else:
            lit = int(rng.integers(1, 4))
            q[i:i + lit] = rng.choice([-2, -1, 1, 2, 70, -9000], size=min(lit, n - i))
            i += lit + int(rng.integers(8, 13))
    return q


@pytest.mark.parametrize("variant", ["dense", "long_literals", "all_dense_small"])
def test_many_token_streams_parallel_parse(cuda, ref, variant):
    """Streams with 10^5-10^6 tokens go through the parallel token parse
    (stream.cu k_tok_jump/resolve/walk); payloads and decodes must match the
    reference byte for byte (lossless.hpp:53-70)."""
    rng = np.random.default_rng({"dense": 1, "long_literals": 2, "all_dense_small": 3}[variant])
    n = 1_500_000 if variant != "all_dense_small" else 40_000
    q = _token_dense_codes(rng, n, long_lits=variant == "long_literals")
    tau = 0.5
    v = q.astype(np.float64) * (2 * tau)
    got = umcg.encode(dev(v), predictor=0, tau=tau)
    want = ref.encode(v, predictor=0, tau=tau)
    assert got == want
    back = umcg.decode(want).cpu().numpy()
    assert np.array_equal(back, v)


def test_many_token_streams_corruption_matches_reference(cuda, ref):
    """Byte flips anywhere in a token-dense stream: the GPU decoder fails with
    corrupt_payload exactly when the reference fails, else decodes the same
    values (the parallel parse falls back to the serial walk on a broken
    chain)."""
    rng = np.random.default_rng(9)
    n = 400_000
    q = _token_dense_codes(rng, n)
    v = q.astype(np.float64)
    pl = ref.encode(v, predictor=0, tau=0.5)
    hdr = 21 + 8 + 8  # 1-D header + escape count (codec.hpp:231-250)
    for trial in range(24):
        b = bytearray(pl)
        pos = int(rng.integers(hdr, len(b)))
        b[pos] = int(rng.choice([0x00, 0x01, 0x05, 0x80, 0xFF, int(rng.integers(0, 256))]))
        b = bytes(b)
        try:
            r = ref.decode(b, n)
            r_err = None
        except Exception as e:  # noqa: BLE001
            r, r_err = None, e
        try:
            g = umcg.decode(b, n_capacity=n).cpu().numpy()
            g_err = None
        except umcg.UmcgError as e:
            g, g_err = None, e
        if r_err is not None:
            assert g_err is not None and g_err.kind == "corrupt_payload", (trial, pos, r_err)
        else:
            assert g_err is None, (trial, pos, g_err)
            assert np.array_equal(g, r), (trial, pos)


@pytest.mark.parametrize("tau", [1e-2, 1e-4])
def test_config3_at_scale_matches_reference(cuda, ref, oracle, tau):
    """BASELINE config 3 (jittered 3-D lattice, Feistel-permuted vertex order)
    at lattice 128 (2.1M vertices, grid 64): the GPU archive against the
    reference's on the same mapping (byte-exact up to rounding-window codes),
    both decoders, and the bound on every vertex. tau=1e-2 gives a stream with
    ~10^5 tokens (parallel token parse)."""
    import torch
    xyz, x = umcg.gen_config(3, 128, 20250113, device="cuda")
    axes = [np.linspace(0.0, 1.0, 64) for _ in range(3)]
    plan = umcg.Plan.build(axes, xyz)
    mode, gaxes, assign, visited = plan.export()
    s = Setup(dim=3, axes=gaxes, mode=mode, assignments=assign, visited=visited)
    xh = x.cpu().numpy()
    b = umcg.Budget(tau=tau, split_rho=0.5, bound_kind=1)
    got = plan.compress(x, b, name="c3")
    want = ref.compress(s, xh, name="c3", tau=tau)
    check_archive(got, want, s, xh, dict(tau=tau), oracle, f"config3 tau={tau}")
    tau_abs = tau * np.ptp(xh)
    out = plan.decompress(got).cpu().numpy()
    check_decode(out, ref.decompress(s, got), xh, tau_abs, "own archive")
    out_r = plan.decompress(want).cpu().numpy()
    check_decode(out_r, ref.decompress(s, want), xh, tau_abs, "ref archive")
    del torch


def test_host_pipeline_matches_sequential_calls(cuda):
    """HostPipeline (compress workers on one or two plans overlapping the
    decompress of earlier fields on another plan of the same mesh, one host
    thread per plan, per-thread streams; pageable and pinned archive slots)
    yields exactly the archives and fields of one-at-a-time calls."""
    import torch
    xyz, x = umcg.gen_config(3, 96, 7, device="cuda")
    axes = [np.linspace(0.0, 1.0, 48) for _ in range(3)]
    pc = umcg.Plan.build(axes, xyz)
    pc2, pd, pd2 = umcg.Plan.build(axes, xyz), pc.clone(), pc.clone()  # a second build and two clones
    assert pd.digest == pc.digest and pd.n == pc.n
    rng = np.random.default_rng(3)
    xs = [x.cpu().numpy() * (1.0 + 0.1 * k) + rng.normal(0, 1e-3, x.numel()) for k in range(7)]
    b = umcg.Budget(tau=1e-3, split_rho=0.5, bound_kind=1)
    cap = pc.compress_bound("f")
    slots = [np.empty(cap, np.uint8) for _ in range(4)]  # pageable: copy-engine uploads
    pinned = [torch.empty(cap, dtype=torch.uint8, pin_memory=True).numpy() for _ in range(4)]  # SM reads
    ref = [pc.compress_host(xs[k], b, "f") for k in range(7)]
    for pcs, pds, sl in (([pc], [pd], slots[:2]), ([pc, pc2], [pd], slots[:3]), ([pc, pc2], [pd, pd2], pinned)):
        outs = [np.empty(x.numel()) for _ in range(7)]
        pipe = umcg.HostPipeline(pcs, pds, sl)
        lens = pipe.run(xs, b, outs, "f")
        lens2 = pipe.run(xs[:3], b, outs[:3], "f")  # workers are reused
        pipe.close()
        assert lens2 == lens[:3]
        for k in range(7):
            assert lens[k] == len(ref[k])
            assert np.array_equal(outs[k], pd.decompress_host(ref[k])), k
    with pytest.raises(ValueError):
        umcg.HostPipeline([pc], pc, slots)
    with pytest.raises(ValueError):
        umcg.HostPipeline([pc, pc2], pd, slots[:2])


def test_plan_clone_lifetime_and_concurrency(cuda):
    """umcg_plan_clone: clones share the mapping arrays, outlive their origin,
    and concurrent calls on different handles give the single-handle bytes."""
    import threading
    xyz, x = umcg.gen_config(3, 64, 11, device="cuda")
    p = umcg.Plan.build([np.linspace(0.0, 1.0, 32) for _ in range(3)], xyz)
    b = umcg.Budget(tau=1e-4)
    ref = p.compress(x, b)
    c1 = p.clone()
    c2 = c1.clone()  # clone of a clone: same origin
    del p  # origin handle destroyed first
    import gc
    gc.collect()
    res = {}

    def work(k, h):
        res[k] = [h.compress(x, b) for _ in range(3)]

    ts = [threading.Thread(target=work, args=(k, h)) for k, h in enumerate((c1, c2))]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert all(a == ref for v in res.values() for a in v)
    assert np.array_equal(c2.decompress(ref).cpu().numpy(), c1.decompress(ref).cpu().numpy())


@pytest.mark.parametrize("tau", [1e-1, 1e-2, 1e-4, 1e-7])
def test_config3_full_size_properties(cuda, tau):
    """Config 3 at the bench size (512^3 vertices, grid 256): size-independent
    properties -- the bound on 100% of vertices, determinism, host path ==
    device path -- across the tau range (1e-1: dense token streams)."""
    import torch
    xyz, x = umcg.gen_config(3, 512, 20250113, device="cuda")
    axes = [np.linspace(0.0, 1.0, 256) for _ in range(3)]
    plan = umcg.Plan.build(axes, xyz)
    del xyz
    b = umcg.Budget(tau=tau, split_rho=0.5, bound_kind=1)
    a1 = plan.compress(x, b)
    a2 = plan.compress(x, b)
    assert a1 == a2
    fb0 = umcg.serial_fallbacks()
    out = plan.decompress(a1)
    assert umcg.serial_fallbacks() == fb0
    rng = float((x.max() - x.min()).item())
    err = (out - x).abs().max().item()
    assert err <= tau * rng, (err, tau * rng)
    torch.cuda.synchronize()


@pytest.mark.parametrize("seed", range(5))
def test_rle_raw_bytes_match_reference(cuda, ref, seed):
    """umcg_rle_compress / umcg_rle_decompress against rle_compress /
    rle_decompress (lossless.hpp:24-70): empty input, all zeros, bytes >= 0x80,
    zero runs of every length around the 8-byte threshold, sizes across the
    2048-byte tiles (test_lossless.cpp:188-220 cases)."""
    rng = np.random.default_rng(300 + seed)
    cases = [b"", bytes(1000), bytes([0x80] * 9), bytes(7) + b"\xff" + bytes(8)]
    for _ in range(6):
        n = int(rng.choice([1, 17, 2047, 2048, 2049, 30000, 300000]))
        parts, tot = [], 0
        while tot < n:
            if rng.random() < 0.4:
                k = int(rng.choice([1, 6, 7, 8, 9, 15, 100, 5000]))
                parts.append(bytes(k))
            else:
                k = int(rng.integers(1, 40))
                parts.append(rng.integers(0, 256, k, dtype=np.uint8).tobytes())
            tot += k
        cases.append(b"".join(parts)[:n])
    for data in cases:
        want = ref.rle_compress(data)
        assert umcg.rle_compress(data) == want, len(data)
        assert umcg.rle_decompress(want, len(data)) == data
    with pytest.raises(umcg.UmcgError) as e:
        umcg.rle_decompress(b"\x02\x05", 16)
    assert e.value.kind == "corrupt_payload"


def test_verbatim_codec_matches_reference(cuda, ref):
    """Codec id 1 (codec.hpp:240-248, 387-397): payload byte-identical to
    the reference, decode bitwise, and the verbatim error checks."""
    rng = np.random.default_rng(44)
    arrays = [np.zeros(5000), rng.normal(size=20000), np.array([1.0, -0.0, 5e307, 1e-300]),
              np.repeat(rng.normal(size=300), 40)]
    for v in arrays:
        for pred, dims in ((1, None), (0, None)):
            got = umcg.encode(dev(v), predictor=pred, dims=dims, tau=1e-3, codec_id=1)
            want = ref.encode(v, predictor=pred, dims=dims, tau=1e-3, codec_id=1)
            assert got == want
            back = umcg.decode(got).cpu().numpy()
            assert np.array_equal(back.view(np.uint64), v.view(np.uint64))
    pl = bytearray(ref.encode(arrays[1], predictor=1, tau=1e-3, codec_id=1))
    with pytest.raises(umcg.UmcgError) as e:
        umcg.decode(bytes(pl[:-3]), n_capacity=len(arrays[1]))
    assert e.value.kind == "corrupt_payload"


def test_pipeline_verbatim_codec_matches_reference(cuda, ref, oracle):
    """compress(..., codec_id=1): both components verbatim (pipeline.hpp:
    96-110, 140-146). Cluster means and residuals are exact, so the archive
    is byte-identical and the decode bitwise equal to the reference's."""
    params, cases = load_cases()
    for k, s, x, archives in cases[:4]:
        plan = plan_for(s)
        for fill, g in ((0, 0), (1, 0), (0, 1), (1, 1)) if s.mode == 0 else ((0, 0),):
            # verbatim residual bytes pin g itself bit for bit (multilinear included)
            b = umcg.Budget(tau=1e-3, codec_id=1, fill=fill, g_kind=g)
            got = plan.compress(dev(x), b, name="v")
            want = ref.compress(s, x, name="v", tau=1e-3, codec_id=1, fill=fill, g_kind=g)
            assert got == want, (k, fill, g)
            out = plan.decompress(got).cpu().numpy()
            assert np.array_equal(out.view(np.uint64), ref.decompress(s, want).view(np.uint64))


def test_baseline_archive_matches_reference(cuda, ref, oracle):
    """umcg_compress_baseline == serialize_archive(baseline_archive(...))
    (pipeline.hpp:152-176, 214-235): one lorenzo_1d component at the full
    budget, flag 8, no digest; its decode meets the bound."""
    params, cases = load_cases()
    rng = np.random.default_rng(8)
    fields = [cases[0][2], cases[3][2], np.cumsum(rng.normal(size=50000)), np.zeros(1000)]
    for x in fields:
        for tau, bk, codec in ((1e-3, 1, 0), (1e-4, 1, 0), (0.01, 0, 0), (1e-3, 1, 1), (0.0, 1, 0)):
            b = umcg.Budget(tau=tau, bound_kind=bk, codec_id=codec)
            got = umcg.compress_baseline(dev(x), b, name="base")
            want = ref.baseline_archive(x, name="base", tau=tau, bound_kind=bk, codec_id=codec)
            if got != want:
                ga, ra = parse_archive(got), parse_archive(want)
                pred = np.concatenate([[0.0], ref.decode(ra["p1"], len(x))[:-1]])
                check_component(ga["p1"], ra["p1"], x, pred, oracle, f"baseline tau={tau}")
            p1 = parse_archive(want)["p1"]
            out = umcg.decode(p1).cpu().numpy()
            tau_abs = tau * (np.ptp(x) if bk else 1.0)
            check_decode(out, ref.decode(p1, len(x)), x, tau_abs, f"baseline decode tau={tau}")
    with pytest.raises(umcg.UmcgError) as e:
        umcg.compress_baseline(dev(fields[0]), umcg.Budget(tau=-1.0))
    assert e.value.kind == "budget_inadmissible"


def test_lattice_rounding_at_half_integers(cuda, ref):
    """Values on and 1-4 ulp around the quantizer's rounding boundaries
    (v / bin = k + 1/2): the GPU lattice index (multiply by fl(1/bin), exact
    divide inside the ambiguity band) must equal std::round(v / bin) of the
    reference exactly -- predictor none makes every code the lattice index
    itself, so the payloads must be byte-identical."""
    rng = np.random.default_rng(77)
    for tau in (0.05, 1e-3, 0.37e-7, 3.3):
        bin_ = 2 * tau
        k = rng.integers(-2**20, 2**20, 4000).astype(np.float64)
        base = (k + 0.5) * bin_
        vals = [base]
        for s in (1, 2, 3, 4):
            up, dn = base.copy(), base.copy()
            for _ in range(s):
                up = np.nextafter(up, np.inf)
                dn = np.nextafter(dn, -np.inf)
            vals += [up, dn]
        v = np.concatenate(vals)
        got = umcg.encode(dev(v), predictor=0, tau=tau)
        want = ref.encode(v, predictor=0, tau=tau)
        assert got == want, tau


def _bbox_plan(xyz, g):
    """Uniform axes over the vertex bbox (SURVEY 8(d) grid recipe), GPU
    grid_coarsen, and the equivalent oracle Setup."""
    lo = xyz.min(0).values.cpu().numpy()
    hi = xyz.max(0).values.cpu().numpy()
    axes = [np.linspace(lo[d], hi[d], g) for d in range(xyz.shape[1])]
    plan = umcg.Plan.build(axes, xyz)
    mode, gaxes, assign, visited = plan.export()
    s = Setup(dim=xyz.shape[1], axes=gaxes, mode=mode, assignments=assign, visited=visited)
    return plan, s


def _parity_case(plan, s, x_dev, xh, p, ref, oracle, label):
    b = budget_of(p)
    got = plan.compress(x_dev, b, name="c")
    want = ref.compress(s, xh, name="c", tau=p["tau"], rho=p.get("rho", 0.5))
    check_archive(got, want, s, xh, p, oracle, label)
    tau_abs = p["tau"] * np.ptp(xh)
    check_decode(plan.decompress(got).cpu().numpy(), ref.decompress(s, got), xh, tau_abs, label + " own")
    check_decode(plan.decompress(want).cpu().numpy(), ref.decompress(s, want), xh, tau_abs, label + " ref")


@pytest.mark.parametrize("g", [256, 1024])
def test_config2_graded_annulus_matches_reference(cuda, ref, oracle, g):
    """BASELINE config 2 (graded annulus, large clusters) at 2^20 vertices:
    archives against the reference at tau 1e-2 / 1e-4 / 1e-6."""
    xy, x = umcg.gen_config(2, 1 << 20, 20250102, device="cuda")
    plan, s = _bbox_plan(xy, g)
    xh = x.cpu().numpy()
    for tau in (1e-2, 1e-4, 1e-6):
        _parity_case(plan, s, x, xh, dict(tau=tau), ref, oracle, f"config2 g={g} tau={tau} mode={s.mode}")


@pytest.mark.parametrize("g", [64, 128])
def test_config5_shell_matches_reference(cuda, ref, oracle, g):
    """BASELINE config 5 (clustered cylinder shell; seed mode when the
    visited fraction drops under 0.35) at 2^21 vertices: the error split and
    tau sweep of the config (rho 0.1 / 0.9, tau 1e-2 / 1e-5)."""
    xyz, x = umcg.gen_config(5, 1 << 21, 20250105, device="cuda")
    plan, s = _bbox_plan(xyz, g)
    xh = x.cpu().numpy()
    for tau, rho in ((1e-2, 0.1), (1e-5, 0.9), (1e-3, 0.5)):
        _parity_case(plan, s, x, xh, dict(tau=tau, rho=rho), ref, oracle,
                     f"config5 g={g} tau={tau} rho={rho} mode={s.mode}")


def test_config5_error_split_sweep_matches_reference(cuda, ref, oracle):
    """BASELINE config 5's nine error splits between the grid and residual
    components (rho 0.1 .. 0.9) at 2^19 vertices, tau 1e-4, dense and seed
    grids."""
    xyz, x = umcg.gen_config(5, 1 << 19, 20250115, device="cuda")
    xh = x.cpu().numpy()
    for g in (48, 96):
        plan, s = _bbox_plan(xyz, g)
        for rho in np.round(np.arange(0.1, 0.95, 0.1), 1):
            _parity_case(plan, s, x, xh, dict(tau=1e-4, rho=float(rho)), ref, oracle,
                         f"config5 split g={g} rho={rho} mode={s.mode}")


def test_config5_modes_cover_dense_and_seed(cuda):
    """The shell switches the grid builder to seed mode as the grid refines
    (128^3 dense, 256^3 seed at 200M vertices)."""
    xyz, _ = umcg.gen_config(5, 1 << 21, 20250105, device="cuda", values=False)
    modes = {g: _bbox_plan(xyz, g)[0].info.mode for g in (32, 160)}
    assert modes[32] == 0 and modes[160] == 1, modes


@pytest.mark.parametrize("tau", [1e-3, 1e-5])
def test_config4_fp32_batch_matches_reference(cuda, ref, oracle, tau):
    """BASELINE config 4: five fp32 variables in one umcg_compress_batch call
    against five reference compress calls on the widened values
    (SURVEY 8(a) row 16)."""
    m = 1024
    xy, vals = umcg.gen_config(4, m, 20250104, device="cuda")
    plan, s = _bbox_plan(xy, 512)
    archives = plan.compress_batch(vals, umcg.Budget(tau=tau), names=[f"v{k}" for k in range(5)])
    assert len(archives) == 5
    for k in range(5):
        xh = vals[k].double().cpu().numpy()
        want = ref.compress(s, xh, name=f"v{k}", tau=tau)
        check_archive(archives[k], want, s, xh, dict(tau=tau), oracle, f"config4 var{k} tau={tau}")
        out = plan.decompress(archives[k]).cpu().numpy()
        check_decode(out, ref.decompress(s, archives[k]), xh, tau * np.ptp(xh), f"config4 var{k}")
    # batched decompress: fp64 equals the single-archive decodes, fp32 is their RN
    import torch
    both = plan.decompress_batch(archives)
    f32 = plan.decompress_batch(archives, dtype=torch.float32)
    for k in range(5):
        one = plan.decompress(archives[k])
        assert torch.equal(both[k], one)
        assert torch.equal(f32[k], one.float())


@pytest.mark.parametrize("g", [128, 256])
def test_config5_full_size_properties(cuda, g):
    """Config 5 at its full 200M vertices (seed mode at 256^3): bound on every
    vertex, determinism, no serial fallback, across the tau range."""
    import torch
    xyz, x = umcg.gen_config(5, 200_000_000, 20250105, device="cuda")
    lo = xyz.min(0).values.cpu().numpy()
    hi = xyz.max(0).values.cpu().numpy()
    plan = umcg.Plan.build([np.linspace(lo[d], hi[d], g) for d in range(3)], xyz)
    del xyz
    # visited fraction 0.376 at 128^3 (dense), 0.317 at 256^3 (seed)
    print(f"g={g} mode={plan.info.mode} visited={plan.info.visited_fraction:.3f}")
    assert plan.info.mode == (1 if g == 256 else 0)
    torch.cuda.empty_cache()
    rng = float((x.max() - x.min()).item())
    for tau in (1e-2, 1e-6):
        b = umcg.Budget(tau=tau)
        a1 = plan.compress(x, b)
        assert plan.compress(x, b) == a1
        fb0 = umcg.serial_fallbacks()
        out = plan.decompress(a1)
        assert umcg.serial_fallbacks() == fb0
        err = (out - x).abs().max().item()
        assert err <= tau * rng, (g, tau, err, tau * rng)
        del out


@pytest.mark.parametrize("dims", [[300, 200], [64, 48, 40], [1, 500, 3], [7, 1, 9]])
def test_lossless_nd_wavefront_matches_reference(cuda, ref, dims):
    """tau = 0 N-D decode (codec.hpp:276-294, 429-430): the hyperplane
    wavefront reproduces the reference's floating-point Lorenzo chain bit
    for bit, without the one-thread replica."""
    rng = np.random.default_rng(sum(dims))
    n = int(np.prod(dims))
    v = np.cumsum(rng.normal(size=n)).reshape(dims)
    v = (v + 1e-3 * rng.normal(size=dims)).ravel()
    v[::7] = 0.0
    pl = ref.encode(v, predictor=2, dims=dims, tau=0.0)
    assert umcg.encode(dev(v), predictor=2, dims=dims, tau=0.0) == pl
    fb0 = umcg.serial_fallbacks()
    out = umcg.decode(pl).cpu().numpy()
    assert np.array_equal(out.view(np.uint64), v.view(np.uint64))
    assert umcg.serial_fallbacks() == fb0


@pytest.mark.parametrize("g", [6, 12])
def test_heavy_slots_match_reference(cuda, ref, oracle, g):
    """Grids so coarse that single slots hold > 4096 vertices (the bucket
    kernels' one-slot heavy path, partition.cu k_bucket heavy_only) next to
    regular buckets: config-1 lattice at 2^20 vertices."""
    xy, x = umcg.gen_config(1, 1024, 20250101, device="cuda")
    c = xy.cpu().numpy()
    axes = [np.linspace(0.0, 1.0, g) for _ in range(2)]
    idx = [np.clip(np.rint(c[:, d] * (g - 1)), 0, g - 1).astype(np.uint64) for d in range(2)]
    s = Setup(dim=2, axes=axes, mode=0, assignments=idx[0] * np.uint64(g) + idx[1], coords=c)
    plan = plan_for(s)
    counts = np.bincount(s.assignments.astype(np.int64))
    assert counts.max() > 4096
    xh = x.cpu().numpy()
    for tau in (1e-2, 1e-5):
        _parity_case(plan, s, x, xh, dict(tau=tau), ref, oracle, f"heavy g={g} tau={tau}")


def _lattice_mesh(rng, dims, jitter, kind):
    """Jittered lattice with permuted vertex ids and cells: 'tri' (2 per
    quad), 'quad', or 'hex'."""
    idx = np.stack(np.meshgrid(*[np.arange(m) for m in dims], indexing="ij"), -1).reshape(-1, len(dims))
    h = [1.0 / (m - 1) for m in dims]
    xyz = idx * np.array(h) + (rng.uniform(-jitter, jitter, idx.shape) * np.array(h)) * \
        ((idx > 0) & (idx < np.array(dims) - 1))
    perm = rng.permutation(len(xyz))
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    lin = lambda *c: np.ravel_multi_index(c, dims)  # noqa: E731
    if kind in ("tri", "quad"):
        i, j = np.meshgrid(np.arange(dims[0] - 1), np.arange(dims[1] - 1), indexing="ij")
        i, j = i.ravel(), j.ravel()
        a, b, c, d = lin(i, j), lin(i + 1, j), lin(i + 1, j + 1), lin(i, j + 1)
        cells = np.concatenate([np.stack([a, b, c], 1), np.stack([a, c, d], 1)]) if kind == "tri" else \
            np.stack([a, b, c, d], 1)
    else:
        i, j, k = [x.ravel() for x in np.meshgrid(*[np.arange(m - 1) for m in dims], indexing="ij")]
        corners = [lin(i + di, j + dj, k + dk) for dk in (0, 1) for (di, dj) in ((0, 0), (1, 0), (1, 1), (0, 1))]
        cells = np.stack(corners, 1)
    return xyz[perm], inv[cells].astype(np.uint64)


@pytest.mark.parametrize("case", ["tri", "quad", "hex", "tri_gmax", "cloud2", "cloud3", "annulus", "tiny"])
def test_grid_init_matches_reference(cuda, ref, case):
    """umcg_grid_init against umc::grid_init (grid_builder.hpp:201-282):
    cell-edge statistics for tri/quad/hex meshes, the 1-NN point-cloud
    fallback, the g_max percentile loop and its uniform fallback, and a
    collinear (degenerate-axis) cloud -- identical axes."""
    import torch
    rng = np.random.default_rng(hash(case) % 2**32)
    cells, arity, kw = None, 3, {}
    if case in ("tri", "quad", "tri_gmax"):
        xyz, cells = _lattice_mesh(rng, [120, 90], 0.3, "tri" if case != "quad" else "quad")
        arity = 4 if case == "quad" else 3
        if case == "tri_gmax":
            kw = dict(g_max=24, percentile_k=30.0, delta=7.5)
    elif case == "hex":
        xyz, cells = _lattice_mesh(rng, [30, 25, 20], 0.2, "hex")
        arity = 8
    elif case == "cloud2":
        xyz = _lattice_mesh(rng, [300, 300], 0.3, "tri")[0]
    elif case == "cloud3":
        xyz = rng.uniform(0, 1, (60000, 3))
    elif case == "annulus":
        xy, _ = umcg.gen_config(2, 200000, 7, device="cuda", values=False)
        xyz = xy.cpu().numpy()
    else:
        xyz = np.array([[0.0, 0.5], [1.0, 0.5], [0.25, 0.5], [0.7, 0.5]])
    want = ref.grid_init(xyz, cells, arity, **kw)
    d_cells = torch.from_numpy(cells.view(np.int64)).cuda() if cells is not None else None
    got = umcg.grid_init(torch.from_numpy(xyz).cuda(), d_cells, arity, **kw)
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert np.array_equal(a, b), (case, len(a), len(b))


@pytest.mark.parametrize("config,fill", [(2, 0), (5, 0), (5, 1)])
def test_multilinear_offset_field_wide_residuals(cuda, ref, oracle, config, fill):
    """Multilinear g on a dense grid with unvisited nodes and a field far from
    zero (x + 1000). Config-2 annulus at 512^2 (the disc inside r = 0.3 holds
    no vertex) and config-5 cylinder shell at 32^3 (whole rows along the
    fastest axis inside the cylinder are unvisited, though grid_coarsen keeps
    their planes). Unvisited nodes hold 0.0 (fill zero, interp.hpp:56) or stay
    0.0 along whole empty rows (nearest_visited, interp.hpp:78), and
    multilinear_at blends them in (interp.hpp:129), so |K2| reaches ~10^7:
    the narrow int16 residual path must detect it and rerun with int32
    indices (it used to truncate silently). Archive against the reference,
    both decoders, the bound on every vertex, no serial fallback."""
    if config == 2:
        xy, x = umcg.gen_config(2, 1 << 20, 20250102, device="cuda")
        g = 512
    else:
        xy, x = umcg.gen_config(5, 1 << 21, 20250105, device="cuda")
        g = 32
    D = xy.shape[1]
    xy_h = xy.cpu().numpy()
    lo, hi = xy_h.min(0), xy_h.max(0)
    axes = [np.linspace(lo[d], hi[d], g) for d in range(D)]
    plan = umcg.Plan.build(axes, xy, keep_coords=True)
    mode, gaxes, assign, visited = plan.export()
    assert mode == 0 and len(visited) < np.prod([len(a) for a in gaxes])
    s = Setup(dim=D, axes=gaxes, mode=mode, assignments=assign, visited=visited, coords=xy_h)
    xh = x.cpu().numpy() + 1000.0
    p = dict(tau=1e-4, rho=0.5, g_kind=1, fill=fill)
    b = budget_of(p)
    fb0 = umcg.serial_fallbacks()
    got = plan.compress(dev(xh), b, name="offset")
    assert umcg.serial_fallbacks() == fb0
    want = ref.compress(s, xh, name="offset", tau=1e-4, rho=0.5, g_kind=1, fill=fill)
    # the residual component really needs more than int16 lattice indices
    p2 = parse_archive(want)["p2"]
    rec2 = oracle.decode(p2)
    assert np.max(np.abs(rec2)) / (2 * parse_payload(p2, oracle.rle_decompress)["tau"]) > 16384
    check_archive(got, want, s, xh, p, oracle, f"multilinear offset config{config} fill={fill}")
    tau_abs = 1e-4 * np.ptp(xh)
    check_decode(plan.decompress(got).cpu().numpy(), ref.decompress(s, got), xh, tau_abs, "own")
    check_decode(plan.decompress(want).cpu().numpy(), ref.decompress(s, want), xh, tau_abs, "ref")


def test_host_calls_pageable_staging(cuda):
    """Host-buffer calls on pageable numpy arrays large enough for the staged
    copy path (pinned 32 MiB pieces, parallel host memcpy; api.cu
    staged_copy), several pieces per transfer and back-to-back transfers in
    one call: the same archive and field as the device path."""
    import torch
    xyz, x = umcg.gen_config(3, 256, 20250113, device="cuda")
    plan = umcg.Plan.build([np.linspace(0.0, 1.0, 128) for _ in range(3)], xyz)
    b = umcg.Budget(tau=1e-4)
    want = plan.compress(x, b, "f")
    xh = x.cpu().numpy().copy()  # pageable, 134 MB
    for _ in range(2):
        got = plan.compress_host(xh, b, "f")
        assert got == want
        out = np.empty(plan.n)
        plan.decompress_host(got, out=out)
        assert np.array_equal(out, plan.decompress(want).cpu().numpy())
    del torch


def test_fine_bound_zero_runs_at_tile_warp_and_thread_boundaries(cuda, ref, oracle):
    """The fine-bound residual path (tau_rel <= 2.5e-4: run-sorted codes,
    k_rle_tiles_fast summaries with the exact fallback) on zero-code runs
    placed across the summary's seams: runs of 7 / 9 / 17 zeros straddling
    thread (8 codes), warp (256) and ENC tile (2048) boundaries, all-zero
    threads and whole zero tiles, and a partial last tile. Two vertices per
    node in vertex order, so a node whose two values are equal has K2 = 0 on
    both and a stretch of such nodes is a run of 2 m - 1 zero codes after
    the stretch's first (nonzero) code."""
    rng = np.random.default_rng(20251020)
    n = (1 << 20) - 6
    nodes = n // 2
    x = rng.normal(0.0, 1.0, n)

    def zero_run(start, length):  # `length` (odd) zero codes starting at code `start` (odd)
        assert start % 2 == 1 and length % 2 == 1
        a = (start - 1) // 2
        m = (length + 1) // 2
        for k in range(a, a + m):
            x[2 * k + 1] = x[2 * k]

    starts = []
    for w in range(1, 60):  # warp boundaries: runs of 7 / 9 / 17 across 256 w
        b = 256 * w
        ln = (7, 9, 17)[w % 3]
        starts.append((b - ln // 2 - (1 if (b - ln // 2) % 2 == 0 else 0), ln))
    for t in range(64, 160, 3):  # thread boundaries inside warps: 7 / 9 zeros across 8 t
        b = 8 * t + 2048 * 40
        ln = 7 if t % 2 else 9
        starts.append((b - 3 if (b - 3) % 2 else b - 4, ln))
    for tile in (100, 101, 300):  # tile boundaries
        starts.append((2048 * tile - 5, 9))
    starts.append((2048 * 200 + 1, 2 * 2048 + 1))  # whole zero tiles (all-zero threads)
    starts.append((n - 2000 + 1, 1999 - 2))  # a long run into the partial last tile
    for s0, ln in starts:
        zero_run(s0, ln)
    axes = [np.linspace(0.0, 1.0, 5), np.linspace(0.0, 1.0, nodes // 5)]
    assert 5 * (nodes // 5) == nodes
    assign = (np.arange(n, dtype=np.uint64) // np.uint64(2))
    s = Setup(dim=2, axes=axes, mode=0, assignments=assign)
    plan = plan_for(s, coords=False)
    for tau in (1e-4, 2e-4):
        _parity_case(plan, s, dev(x), x, dict(tau=tau), ref, oracle, f"zero-run seams tau={tau}")
