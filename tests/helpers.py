"""Test helpers: golden fixture loading, archive parsing, code-level diffs.

Archive / payload layouts follow the reference byte formats
(pipeline.hpp:214-235, codec.hpp:225-233, lossless.hpp:24-51).
"""
from __future__ import annotations

import os
import struct

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

WINDOW = 1e-6          # rounding-window half width, in bins
REL_TOL = 1e-12        # decode tolerance relative to max(range, max|x|)


def load_cases():
    from oracle.bindings import Setup
    z = np.load(os.path.join(GOLDEN, "cases.npz"))
    params = [eval(p) for p in z["params"]]  # noqa: S307 - our own fixture
    cases = []
    for k in range(int(z["n_setups"])):
        dim = z[f"s{k}_coords"].shape[1]
        s = Setup(dim=dim, axes=[z[f"s{k}_axis{d}"] for d in range(dim)], mode=int(z[f"s{k}_mode"]),
                  assignments=z[f"s{k}_assign"], visited=z[f"s{k}_visited"], coords=z[f"s{k}_coords"])
        archives = [z[f"s{k}_p{j}"].tobytes() for j in range(len(params))]
        cases.append((k, s, z[f"s{k}_values"], archives))
    return params, cases


def load_seed7():
    from oracle.bindings import Setup
    z = np.load(os.path.join(GOLDEN, "seed7_case.npz"))
    s = Setup(dim=2, axes=[z["axis0"], z["axis1"]], mode=int(z["mode"]), assignments=z["assignments"],
              visited=z["visited"], coords=z["coords"])
    with open(os.path.join(GOLDEN, "archive_seed7.umcz"), "rb") as f:
        ar = f.read()
    return s, z["values"], ar


def parse_archive(b: bytes) -> dict:
    assert b[:4] == b"UMCZ"
    ver, flags, nl = struct.unpack_from("<HHH", b, 4)
    o = 10 + nl
    digest, tau, rho, l1 = struct.unpack_from("<QddQ", b, o)
    o += 32
    p1 = b[o:o + l1]
    o += l1
    (l2,) = struct.unpack_from("<Q", b, o)
    o += 8
    p2 = b[o:o + l2]
    return dict(flags=flags, name=b[10:10 + nl].decode(), digest=digest, tau=tau, rho=rho, p1=p1, p2=p2)


def parse_payload(p: bytes, rle_decompress) -> dict:
    codec, pred, backend, _ = p[0], p[1], p[2], p[3]
    tau, n = struct.unpack_from("<dQ", p, 4)
    D = p[20]
    dims = list(struct.unpack_from("<%dQ" % D, p, 21))
    o = 21 + 8 * D
    (ne,) = struct.unpack_from("<Q", p, o)
    o += 8
    esc = np.frombuffer(p[o:o + 16 * ne], dtype=[("i", "<u8"), ("v", "<f8")])
    o += 16 * ne
    stream = p[o:]
    raw = np.frombuffer(rle_decompress(stream), np.uint8)
    codes = varint_decode(raw)
    return dict(codec=codec, pred=pred, backend=backend, tau=tau, n=n, dims=dims, esc=esc,
                stream=stream, codes=codes)


def varint_decode(raw: np.ndarray) -> np.ndarray:
    """ByteReader::varint over a whole byte stream (common.hpp:99-107), vectorised."""
    if raw.size == 0:
        return np.zeros(0, np.uint64)
    ends = np.flatnonzero((raw & 0x80) == 0)
    starts = np.concatenate([[0], ends[:-1] + 1])
    lens = ends - starts + 1
    out = np.zeros(len(ends), np.uint64)
    for k in range(int(lens.max())):
        sel = lens > k
        out[sel] |= (raw[starts[sel] + k].astype(np.uint64) & np.uint64(0x7F)) << np.uint64(7 * k)
    return out


def zz_dec(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64)
    return (z >> np.uint64(1)).astype(np.int64) ^ -(z & np.uint64(1)).astype(np.int64)


def lorenzo_pred(recon: np.ndarray, dims) -> np.ndarray:
    """Reference N-D Lorenzo prediction (codec.hpp:61-80) from reconstructed
    values, vectorised: pred accumulated from 0.0 in mask order."""
    r = recon.reshape(dims)
    D = len(dims)
    pred = np.zeros_like(r)
    for mask in range(1, 1 << D):
        sl_dst, sl_src = [], []
        for d in range(D):
            if (mask >> d) & 1:
                sl_dst.append(slice(1, None))
                sl_src.append(slice(None, -1))
            else:
                sl_dst.append(slice(None))
                sl_src.append(slice(None))
        term = np.zeros_like(r)
        term[tuple(sl_dst)] = r[tuple(sl_src)]
        if bin(mask).count("1") & 1:
            pred = pred + term
        else:
            pred = pred - term
    return pred.ravel()


def window_distance(values: np.ndarray, pred: np.ndarray, tau: float) -> np.ndarray:
    """|frac(t) - 0.5| with t = (v - p_ref)/bin: 0 at a bin boundary."""
    t = (values - pred) / (2.0 * tau)
    return np.abs(t - np.floor(t) - 0.5)


def lattice_k(codes: np.ndarray, pred: int, dims) -> np.ndarray:
    """The lattice index a code stream integrates to: the inclusive prefix of
    the zigzag-decoded codes along the predictor's axes (lorenzo_1d: one
    cumsum; lorenzo_nd: one cumsum per axis, codec.hpp:61-80)."""
    q = zz_dec(codes)
    if pred == 0:
        return q
    if pred == 1 or len(dims) == 1:
        return np.cumsum(q)
    k = q.reshape(dims)
    for ax in range(len(dims)):
        k = np.cumsum(k, axis=ax)
    return k.ravel()


def check_component(gp, rp, values, pred_ref, oracle, label):
    """Byte-exact payload, or the same lattice up to rounding-window events.

    A code that rounds the other way inside the window (|frac(t) - 1/2| <
    WINDOW, t = (v - p_ref) / bin) moves that element's lattice index K by one;
    the following code(s) of the chain compensate, so the integrated lattice
    agrees again right after. The check is therefore on K (the prefix of the
    codes along the predictor): every element whose K differs must differ by
    exactly one and be a window event. Escape records must be identical.
    Returns the number of differing codes."""
    if gp == rp:
        return 0
    g = parse_payload(gp, oracle.rle_decompress)
    r = parse_payload(rp, oracle.rle_decompress)
    for k in ("codec", "pred", "backend", "tau", "n", "dims"):
        assert g[k] == r[k], (label, k)
    assert len(g["esc"]) == len(r["esc"]) and np.array_equal(g["esc"], r["esc"]), label
    assert len(g["codes"]) == len(r["codes"]) == g["n"], label
    bad = np.flatnonzero(g["codes"] != r["codes"])
    assert bad.size > 0, f"{label}: payloads differ but codes agree (stream encoder bug)"
    kg = lattice_k(g["codes"], g["pred"], g["dims"])
    kr = lattice_k(r["codes"], r["pred"], r["dims"])
    kd = np.flatnonzero(kg != kr)
    assert kd.size > 0, (label, "codes differ but integrate to the same lattice", bad[:10])
    assert np.all(np.abs(kg[kd] - kr[kd]) == 1), (label, kd[:10])
    wd = window_distance(values[kd], pred_ref[kd], r["tau"])
    assert np.all(wd < WINDOW), (label, kd[:10], wd[:10])
    return bad.size


def check_archive(gpu_ar, ref_ar, s, x, p, oracle, label):
    """Archive bytes equal, or equal up to codes in the rounding window.
    Returns the number of differing codes per component."""
    if gpu_ar == ref_ar:
        return {"grid": 0, "resid": 0}
    ga, ra = parse_archive(gpu_ar), parse_archive(ref_ar)
    for k in ("flags", "name", "digest", "tau", "rho"):
        assert ga[k] == ra[k], (label, k)
    # component 1: grid, exact cluster means vs reference Lorenzo prediction
    x1 = oracle.interpolate_to_grid(s, x, fill=p.get("fill", 0))
    rec1 = oracle.decode(ra["p1"])
    if s.mode == 1:
        pred1 = np.concatenate([[0.0], rec1[:-1]])
    else:
        pred1 = lorenzo_pred(rec1, list(s.shape))
    d1 = check_component(ga["p1"], ra["p1"], x1, pred1, oracle, label + "/grid")
    # component 2: residuals vs the previous reconstructed residual
    x2 = oracle.residuals(s, x, fill=p.get("fill", 0), g_kind=p.get("g_kind", 0))
    rec2 = oracle.decode(ra["p2"])
    pred2 = np.concatenate([[0.0], rec2[:-1]])
    d2 = check_component(ga["p2"], ra["p2"], x2, pred2, oracle, label + "/resid")
    return {"grid": d1, "resid": d2}


def check_decode(out, ref_out, x, tau_abs, label):
    """GPU decode within REL_TOL * max(range, max|x|) of the reference's decode
    and within the bound of x. Returns (drift / scale, max error / tau_abs)."""
    scale = max(float(np.ptp(x)) if x.size else 0.0, float(np.abs(x).max()) if x.size else 0.0, 1e-300)
    if tau_abs == 0.0:
        assert np.array_equal(out.view(np.uint64), ref_out.view(np.uint64)), label
        return 0.0, 0.0
    drift = float(np.max(np.abs(out - ref_out))) if out.size else 0.0
    err = float(np.max(np.abs(out - x))) if out.size else 0.0
    assert drift <= REL_TOL * scale, (label, drift)
    assert err <= tau_abs, (label, err, tau_abs)
    return drift / scale, err / tau_abs
