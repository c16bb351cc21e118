"""Test helpers: golden fixture loading, archive parsing, code-level diffs.

Archive / payload layouts follow the reference byte formats
(pipeline.hpp:214-235, codec.hpp:225-233, lossless.hpp:24-51).
"""
from __future__ import annotations

import os
import struct

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


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
