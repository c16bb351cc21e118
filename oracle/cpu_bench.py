"""TEST / BENCH INFRASTRUCTURE ONLY: the CPU reference arm.

Times the unmodified reference (oracle/_ref/libumcref.so: umc::compress +
serialize_archive, deserialize_archive + umc::decompress, pipeline.hpp:117-148,
180-210) on the BASELINE config-3 workload built entirely on the host:

* inputs from the host generator (oracle/datagen_host.c), byte-identical to
  the GPU arm's device-generated field;
* the mapping from the reference's own grid_coarsen (grid_builder.hpp:365)
  over the same uniform 256^3 axes the GPU arm uses;
* no import of the product package: this process loads only
  oracle/_ref/libumcref.so (the reference behind its shim, plus the host
  generator compiled into the same library).

A sample is a block of the full 512^3 lattice (lattice points with every
index below `block`, kept in the full mesh's permuted vertex order): exactly
the vertices, coordinates and field values the full-size run has there, and
the same vertex-per-node density (the reference's grid_coarsen deletes the
grid planes the block does not reach). `block=512` is the full workload.

Run as a module to print one JSON line (the single-core baseline; the
timed calls are pinned to one CPU after the multi-threaded input generation):
    python -m oracle.cpu_bench --block 256 --reps 3 --pin 1
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
if os.path.dirname(HERE) not in sys.path:
    sys.path.insert(0, os.path.dirname(HERE))

from oracle.bindings import REF_SO, HostGen, Ref  # noqa: E402

LATTICE, GRID = 512, 256
SEED = 0x250106910 + 3


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def host_info() -> dict:
    aff = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else []
    return {"nproc": os.cpu_count(), "affinity_cpus": len(aff), "cpu_model": cpu_model()}


def build_sample(block: int, gen_threads: int | None = None):
    """(ref, ctx, setup, x) for the config-3 block sample, host-only (the
    generator exported by oracle/_ref/libumcref.so itself: this process loads
    nothing outside oracle/_ref)."""
    g = HostGen(path=REF_SO, threads=gen_threads)
    t0 = time.perf_counter()
    if block >= LATTICE:
        xyz, x = g.gen(3, LATTICE, SEED)
    else:
        xyz, x = g.gen3_block(LATTICE, SEED, [0, 0, 0], [block] * 3)
    t_gen = time.perf_counter() - t0
    R = Ref()
    axes = [np.linspace(0.0, 1.0, GRID) for _ in range(3)]
    t0 = time.perf_counter()
    s, frac = R.grid_coarsen(3, xyz, axes)
    t_map = time.perf_counter() - t0
    s.coords = None  # nearest g never reads vertex coordinates (interp.hpp:153-156)
    del xyz
    ctx = R.ctx(s)
    info = {"vertices": int(x.size), "grid": [len(a) for a in s.axes], "mode": "seed" if s.mode else "dense",
            "visited_fraction": frac, "gen_s": t_gen, "grid_coarsen_s": t_map}
    return R, ctx, s, x, info


def time_digest(R: Ref, ctx, reps: int = 3) -> float:
    """mapping_digest (serialize.hpp:300): charged once per compress and once
    per decompress call by the reference (pipeline.hpp:135, 188)."""
    import ctypes as C
    d = C.c_uint64()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        R._check(R.lib.umcref_mapping_digest(ctx.h, C.byref(d)))
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def single_core(block: int, reps: int, tau: float, pin: int | None = None) -> dict:
    """Median of `reps` compress / decompress calls on the calling thread.
    pin: after the (multi-threaded) input generation, restrict the process to
    that one CPU (sched_setaffinity, what `taskset -c` does) for the timed
    calls."""
    R, ctx, s, x, info = build_sample(block)
    if pin is not None:
        os.sched_setaffinity(0, {pin})
    tc, td = [], []
    ab = 0
    for _ in range(reps):
        c, d, ab = R.time_roundtrip(ctx, x, tau, reps=1)
        tc.append(c)
        td.append(d)
    dig = time_digest(R, ctx)
    mc, md = statistics.median(tc), statistics.median(td)
    nbytes = x.size * 8
    return dict(info, **host_info(), kind="reference", cores=1, reps=reps, tau_rel=tau, archive_bytes=ab,
                compress_s=mc, decompress_s=md, compress_all_s=tc, decompress_all_s=td, digest_s=dig,
                compress_gbs=nbytes / mc / 1e9, decompress_gbs=nbytes / md / 1e9,
                roundtrip_gbs=nbytes / (mc + md) / 1e9,
                roundtrip_gbs_minus_digest=nbytes / (mc + md - 2 * dig) / 1e9)


class Concurrent:
    """`threads` concurrent reference round trips on one sample per step (the
    reference is reentrant; each call is single-threaded)."""

    def __init__(self, block: int, threads: int, tau: float):
        self.R, self.ctx, self.s, self.x, self.info = build_sample(block)
        self.threads, self.tau = threads, tau
        self.per_call = []

    def step(self) -> float:
        res = []

        def work():
            res.append(self.R.time_roundtrip(self.ctx, self.x, self.tau, reps=1))

        ts = [threading.Thread(target=work) for _ in range(self.threads)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        dt = time.perf_counter() - t0
        self.per_call += res
        return dt


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--block", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tau", type=float, default=1e-4)
    ap.add_argument("--pin", type=int, default=None, help="CPU to pin the timed calls to")
    a = ap.parse_args()
    print(json.dumps(single_core(a.block, a.reps, a.tau, a.pin)))
    return 0


if __name__ == "__main__":
    sys.exit(main())
