"""Regenerate the golden fixtures in tests/golden/ from the UNMODIFIED
reference (oracle/_ref/libumcref.so, compiled from /root/reference headers by
oracle/Makefile). Run in the build container (needs /root/reference):

    make -C oracle && python tests/golden/make_golden.py

Outputs (all small, committed):
  grid_seed7.umcg / map_seed7.umcp / archive_seed7.umcz
      the reference's own golden images (tests/support/golden_recipe.hpp:22-45,
      gen_golden.cpp); sha256 recorded in SURVEY.md 8(c).
  seed7_case.npz     mesh coords + field + mapping of that recipe.
  cases.npz          pipeline cases: setups, fields and reference archives over
                     dense/seed mode, nearest/multilinear g, zero/nearest fill,
                     tau sweep incl. tau = 0.
  codec.npz          component-codec known answers (test_codec.cpp cases).
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle.bindings import Ref  # noqa: E402


def main():
    R = Ref()
    g, m, a = R.make_golden(7)
    for name, b in [("grid_seed7.umcg", g), ("map_seed7.umcp", m), ("archive_seed7.umcz", a)]:
        with open(os.path.join(HERE, name), "wb") as f:
            f.write(b)
        print(name, len(b), hashlib.sha256(b).hexdigest())
    s, x = R.build_case(2, 3000, 2, 2, 7)  # holed, white noise: the golden recipe
    np.savez_compressed(os.path.join(HERE, "seed7_case.npz"), coords=s.coords, values=x,
                        axis0=s.axes[0], axis1=s.axes[1], mode=s.mode,
                        assignments=s.assignments, visited=s.visited)

    # pipeline cases: (dim, n_target, mesh_style, field_kind, seed)
    specs = [(2, 4000, 0, 0, 11), (2, 6000, 1, 1, 12), (2, 3000, 2, 2, 13), (3, 8000, 0, 0, 14),
             (3, 6000, 1, 1, 15)]
    params = [dict(tau=1e-2), dict(tau=1e-4), dict(tau=1e-6), dict(tau=0.0),
              dict(tau=1e-3, g_kind=1), dict(tau=1e-3, fill=1), dict(tau=0.05, bound_kind=0, rho=0.3)]
    out = {}
    k = 0
    for (dim, nt, ms, fk, seed) in specs:
        s, x = R.build_case(dim, nt, ms, fk, seed)
        out[f"s{k}_coords"] = s.coords
        out[f"s{k}_values"] = x
        for d in range(dim):
            out[f"s{k}_axis{d}"] = s.axes[d]
        out[f"s{k}_mode"] = np.array(s.mode)
        out[f"s{k}_assign"] = s.assignments
        out[f"s{k}_visited"] = s.visited
        for j, p in enumerate(params):
            try:
                ar = R.compress(s, x, name=f"case{k}", **p)
            except Exception as e:  # seed mode + multilinear -> seed_mode_unsupported
                ar = ("ERR:" + str(e)).encode()
            out[f"s{k}_p{j}"] = np.frombuffer(ar, np.uint8)
        print("case", k, "dim", dim, "n", s.n_v, "mode", s.mode, "shape", s.shape)
        k += 1
    # explicit uniform grids over permuted jittered lattices (the BASELINE
    # config 1 / 3 construction at small size): dense 2D and dense 3D
    rng = np.random.default_rng(99)
    for dim, m, gsz in [(2, 160, 48), (3, 28, 12)]:
        h = 1.0 / (m - 1)
        idx = np.stack(np.meshgrid(*([np.arange(m)] * dim), indexing="ij"), -1).reshape(-1, dim)
        jit = (rng.uniform(-0.25, 0.25, idx.shape) * h) * ((idx > 0) & (idx < m - 1))
        coords = idx * h + jit
        coords = coords[rng.permutation(len(coords))]
        axes = [np.linspace(0.0, 1.0, gsz) for _ in range(dim)]
        s, frac = R.grid_coarsen(dim, coords, axes)
        x = np.sin(4 * np.pi * coords[:, 0]) * np.cos(3 * np.pi * coords[:, 1]) + 0.3 * coords[:, -1] ** 2
        out[f"s{k}_coords"] = s.coords
        out[f"s{k}_values"] = x
        for d in range(dim):
            out[f"s{k}_axis{d}"] = s.axes[d]
        out[f"s{k}_mode"] = np.array(s.mode)
        out[f"s{k}_assign"] = s.assignments
        out[f"s{k}_visited"] = s.visited
        for j, p in enumerate(params):
            try:
                ar = R.compress(s, x, name=f"case{k}", **p)
            except Exception as e:
                ar = ("ERR:" + str(e)).encode()
            out[f"s{k}_p{j}"] = np.frombuffer(ar, np.uint8)
        print("case", k, "dim", dim, "n", s.n_v, "mode", s.mode, "shape", s.shape, "frac", frac)
        k += 1
    out["n_setups"] = np.array(k)
    out["params"] = np.array([repr(p) for p in params])
    np.savez_compressed(os.path.join(HERE, "cases.npz"), **out)

    # codec known answers (reference tests/test_codec.cpp)
    c = {}
    c["worked_in"] = np.array([0.37])
    c["worked_payload"] = np.frombuffer(R.encode([0.37], predictor=0, tau=0.05), np.uint8)
    esc = np.array([1e300 if i % 2 else -1e300 for i in range(500)])
    c["esc_in"] = esc
    c["esc_payload"] = np.frombuffer(R.encode(esc, predictor=1, tau=1e-12), np.uint8)
    rng = np.random.default_rng(2)
    v = rng.uniform(-1e9, 1e9, 4000)
    v[7], v[8], v[9] = 1e-300, -0.0, 5e307
    c["lossless_in"] = v
    c["lossless_payload1"] = np.frombuffer(R.encode(v, predictor=1, tau=0.0), np.uint8)
    c["lossless_payload0"] = np.frombuffer(R.encode(v, predictor=0, tau=0.0), np.uint8)
    z = np.zeros(10000)
    for t in (0.0, 1e-6, 0.5):
        c[f"zeros_payload_{t}"] = np.frombuffer(R.encode(z, predictor=1, tau=t), np.uint8)
    walk = np.cumsum(rng.uniform(-1e-3, 1e-3, 100000))
    c["walk_in"] = walk
    c["walk_payload"] = np.frombuffer(R.encode(walk, predictor=1, tau=1e-3), np.uint8)
    grid = rng.uniform(-50, 50, (17, 9, 5)).cumsum(axis=0).ravel() * 0.01
    c["nd_in"] = grid
    c["nd_payload"] = np.frombuffer(R.encode(grid, predictor=2, dims=[17, 9, 5], tau=1e-3), np.uint8)
    c["nd0_payload"] = np.frombuffer(R.encode(grid, predictor=2, dims=[17, 9, 5], tau=0.0), np.uint8)
    sm = np.sin(np.arange(20000) * 0.001) * 10.0
    c["smooth_in"] = sm
    for t in (1e-6, 1e-5, 1e-4, 1e-3, 1e-2):
        c[f"smooth_payload_{t}"] = np.frombuffer(R.encode(sm, predictor=1, tau=t), np.uint8)
    np.savez_compressed(os.path.join(HERE, "codec.npz"), **c)
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
