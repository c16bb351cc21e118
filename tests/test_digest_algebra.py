"""CPU check of the algebra behind the device mapping digest (csrc/digest.cu).

FNV-1a is h <- (h ^ b) * P. The XOR touches only the low byte l of h, so over
any byte range the hash leaving it is P^len * h_in + B_s (mod 2^64), where s is
the low byte of the hash entering it and B follows B <- (B + ((l ^ b) - l)) * P
along the 256-state trajectory l <- ((l ^ b) * (P mod 256)) mod 256. This test
evaluates exactly that chunk-wise form (records of 8 little-endian bytes, the
high zero bytes as one multiplication) and compares it with the oracle's
mapping_digest (serialize.hpp:255-267, 300-303) on a dense and a seed mapping.
"""
import numpy as np
import pytest

from oracle.bindings import Oracle, Setup

M = (1 << 64) - 1
P = 0x100000001B3
H0 = 0xCBF29CE484222325


def fnv_bytes(h, data):
    for b in data:
        h = ((h ^ b) * P) & M
    return h


def chunk_map(records, s):
    """B_s of a chunk of u64 records for the entry low byte s."""
    l, B = s, 0
    for v in records:
        v = int(v)
        hb = (v.bit_length() + 7) // 8
        for k in range(hb):
            t = l ^ ((v >> (8 * k)) & 0xFF)
            B = ((B + (t - l)) * P) & M
            l = (t * 0xB3) & 0xFF
        B = (B * pow(P, 8 - hb, 1 << 64)) & M
        l = (l * pow(0xB3, 8 - hb, 256)) & 0xFF
    return B


def fnv_records(h, records, chunk):
    for c in range(0, len(records), chunk):
        part = records[c:c + chunk]
        h = (pow(P, 8 * len(part), 1 << 64) * h + chunk_map(part, h & 0xFF)) & M
    return h


def digest(mode, assign, visited, chunk):
    h = fnv_bytes(H0, b"UMCP" + (1).to_bytes(2, "little") + bytes([mode]) + len(assign).to_bytes(8, "little"))
    h = fnv_records(h, assign, chunk)
    if mode == 1:
        h = fnv_bytes(h, len(visited).to_bytes(8, "little"))
        h = fnv_records(h, visited, chunk)
    return h


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("chunk", [1, 7, 64])
def test_chunked_fnv_matches_oracle_digest(mode, chunk):
    rng = np.random.default_rng(7 + mode)
    g = 40
    axes = [np.linspace(0.0, 1.0, g), np.linspace(0.0, 1.0, g)]
    n = 333
    if mode == 0:
        a = rng.integers(0, g * g, n).astype(np.uint64)
        a[::5] = 0
        s = Setup(2, axes, 0, a)
        vis = np.zeros(0, np.uint64)
    else:
        vis = np.sort(rng.choice(g * g, 97, replace=False)).astype(np.uint64)
        a = rng.integers(0, len(vis), n).astype(np.uint64)
        s = Setup(2, axes, 1, a, vis)
    assert digest(mode, a, vis, chunk) == Oracle().mapping_digest(s)
