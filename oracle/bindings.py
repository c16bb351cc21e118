"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the two CPU oracles.

* ``Ref``    -- oracle/_ref/libumcref.so: the unmodified reference library
               (header-only C++20 from /root/reference/proj/include) behind
               the extern "C" shim in oracle/ref_shim.cpp.
* ``Oracle`` -- oracle/liboracle.so: the plain-C restatement (umc_oracle.c).
* ``HostGen`` -- oracle/libdatagen_host.so: the host generator of the
               synthetic BASELINE inputs, byte-identical to the device one.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg (and
its ``--impl reference`` arm) may import this module, and only as the checker
or the reported CPU baseline -- never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libumcref.so")
ORACLE_SO = os.path.join(HERE, "liboracle.so")
DATAGEN_SO = os.path.join(HERE, "libdatagen_host.so")

u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)

# Same numbering as include/umcg.h (umcg_status) and common.hpp:19-38.
ERROR_NAMES = {
    1: "error", 2: "malformed_file", 3: "index_out_of_range", 4: "non_finite_value",
    5: "io_failure", 6: "degenerate_mesh", 7: "empty_after_filtering",
    8: "internal_inconsistency", 9: "seed_mode_unsupported", 10: "unknown_codec",
    11: "corrupt_payload", 12: "external_codec_violation", 13: "subprocess_failure",
    14: "budget_inadmissible", 15: "mapping_mismatch", 16: "zero_norm_reference",
    17: "mismatched_runs", 99: "std_exception",
}


class OracleError(Exception):
    def __init__(self, kind: int, msg: str):
        super().__init__(f"{ERROR_NAMES.get(kind, kind)}: {msg}")
        self.kind = kind
        self.name = ERROR_NAMES.get(kind, str(kind))


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


@dataclass
class Setup:
    """A grid + mapping (+ optional coordinates): the static inputs of the path."""
    dim: int
    axes: list  # list of 1-D float64 arrays
    mode: int  # 0 dense, 1 seed
    assignments: np.ndarray  # uint64 [n_v]
    visited: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    coords: np.ndarray | None = None  # float64 [n_v, dim]

    @property
    def n_v(self) -> int:
        return int(self.assignments.shape[0])

    @property
    def shape(self):
        return tuple(len(a) for a in self.axes)

    @property
    def n1(self) -> int:
        return int(len(self.visited)) if self.mode == 1 else int(np.prod(self.shape))

    def axis_arrays(self):
        sizes = np.array([len(a) for a in self.axes], dtype=np.uint64)
        cat = np.ascontiguousarray(np.concatenate([np.asarray(a, np.float64) for a in self.axes]))
        return sizes, cat


class _Oracle(C.Structure):
    _fields_ = [("dim", C.c_int), ("axis_sizes", u64p), ("axes", f64p), ("mode", C.c_int),
                ("n_v", C.c_uint64), ("assignments", u64p), ("n_visited", C.c_uint64),
                ("visited", u64p), ("coords", f64p)]


class _OParams(C.Structure):
    _fields_ = [("tau", C.c_double), ("rho", C.c_double), ("coeff_abs_sum", C.c_double),
                ("bound_kind", C.c_int), ("g_kind", C.c_int), ("fill", C.c_int)]


def _bytes_out(lib, p, n):
    b = C.string_at(p, n.value) if n.value else b""
    lib.free(p)
    return b


class Ref:
    """The unmodified reference (oracle/_ref/libumcref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        self.lib = L = C.CDLL(path)
        L.umcref_last_error.restype = C.c_char_p
        L.umcref_ctx_create.restype = C.c_void_p
        L.umcref_ctx_create.argtypes = [C.c_int, u64p, f64p, C.c_int, C.c_uint64, u64p,
                                        C.c_uint64, u64p, C.c_int, f64p]
        L.umcref_ctx_destroy.argtypes = [C.c_void_p]
        L.umcref_free.argtypes = [C.c_void_p]
        L.umcref_compress_ctx.argtypes = [C.c_void_p, f64p, C.c_uint64, C.c_char_p, C.c_double,
                                          C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                                          C.c_int, C.c_int, C.POINTER(u8p), u64p]
        L.umcref_decompress_ctx.argtypes = [C.c_void_p, u8p, C.c_uint64, f64p, C.c_uint64, u64p]
        L.umcref_time_roundtrip.argtypes = [C.c_void_p, f64p, C.c_uint64, C.c_double,
                                            C.c_double, C.c_int, C.c_int, f64p, f64p, u64p]
        L.umcref_encode.argtypes = [f64p, C.c_uint64, C.c_int, C.c_int, u64p, C.c_double,
                                    C.c_int, C.c_int, C.POINTER(u8p), u64p]
        L.umcref_decode.argtypes = [u8p, C.c_uint64, f64p, C.c_uint64, u64p]
        L.umcref_rle_compress.argtypes = [u8p, C.c_uint64, C.POINTER(u8p), u64p]
        L.umcref_rle_decompress.argtypes = [u8p, C.c_uint64, C.POINTER(u8p), u64p]
        L.umcref_split_budget.argtypes = [C.c_double, C.c_double, C.c_double, f64p, f64p]
        L.umcref_interpolate_to_grid.argtypes = [C.c_void_p, f64p, C.c_uint64, C.c_int, f64p,
                                                 C.c_uint64, u64p]
        L.umcref_mapping_digest.argtypes = [C.c_void_p, u64p]
        L.umcref_grid_coarsen.argtypes = [C.c_int, C.c_uint64, f64p, u64p, f64p, C.c_double,
                                          u64p, C.POINTER(f64p), C.POINTER(C.c_int),
                                          C.POINTER(u64p), u64p, C.POINTER(u64p), f64p]
        L.umcref_build_case.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_uint64, u64p,
                                        C.POINTER(f64p), C.POINTER(f64p), u64p, C.POINTER(f64p),
                                        C.POINTER(C.c_int), C.POINTER(u64p), u64p,
                                        C.POINTER(u64p)]
        L.umcref_make_golden.argtypes = [C.c_uint64, C.POINTER(u8p), u64p, C.POINTER(u8p), u64p,
                                         C.POINTER(u8p), u64p]
        L.umcref_serialize_mapping.argtypes = [C.c_void_p, C.POINTER(u8p), u64p]
        L.umcref_serialize_grid.argtypes = [C.c_int, u64p, f64p, C.POINTER(u8p), u64p]
        self.free = L.umcref_free

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.umcref_last_error().decode())

    # -- context ------------------------------------------------------------
    def ctx(self, s: Setup):
        sizes, cat = s.axis_arrays()
        a = np.ascontiguousarray(s.assignments, np.uint64)
        v = np.ascontiguousarray(s.visited, np.uint64)
        coords = None if s.coords is None else np.ascontiguousarray(s.coords, np.float64)
        h = self.lib.umcref_ctx_create(s.dim, _ptr(sizes, u64p), _ptr(cat, f64p), s.mode, s.n_v,
                                       _ptr(a, u64p), len(v), _ptr(v, u64p), s.dim,
                                       _ptr(coords, f64p))
        return _Ctx(self, h)

    def compress(self, s: Setup, x, name="x", tau=1e-3, rho=0.5, bound_kind=1, g_kind=0,
                 coeff_abs_sum=1.0, fill=0, codec_id=0, backend_id=0, ctx=None) -> bytes:
        c = ctx or self.ctx(s)
        x = np.ascontiguousarray(x, np.float64)
        p, n = u8p(), C.c_uint64()
        rc = self.lib.umcref_compress_ctx(c.h, _ptr(x, f64p), len(x), name.encode(), tau, rho,
                                          bound_kind, g_kind, coeff_abs_sum, fill, codec_id,
                                          backend_id, C.byref(p), C.byref(n))
        self._check(rc)
        return _bytes_out(self, p, n)

    def decompress(self, s: Setup, archive: bytes, ctx=None) -> np.ndarray:
        c = ctx or self.ctx(s)
        out = np.empty(max(s.n_v, 1), np.float64)
        buf = np.frombuffer(archive, np.uint8)
        n = C.c_uint64()
        rc = self.lib.umcref_decompress_ctx(c.h, _ptr(buf, u8p), len(buf), _ptr(out, f64p),
                                            len(out), C.byref(n))
        self._check(rc)
        return out[: n.value]

    def time_roundtrip(self, ctx, x, tau, rho=0.5, bound_kind=1, reps=1):
        x = np.ascontiguousarray(x, np.float64)
        tc, td, ab = C.c_double(), C.c_double(), C.c_uint64()
        rc = self.lib.umcref_time_roundtrip(ctx.h, _ptr(x, f64p), len(x), tau, rho, bound_kind,
                                            reps, C.byref(tc), C.byref(td), C.byref(ab))
        self._check(rc)
        return tc.value, td.value, ab.value

    def interpolate_to_grid(self, s: Setup, x, fill=0) -> np.ndarray:
        c = self.ctx(s)
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(max(s.n1, 1), np.float64)
        n = C.c_uint64()
        self._check(self.lib.umcref_interpolate_to_grid(c.h, _ptr(x, f64p), len(x), fill,
                                                        _ptr(out, f64p), len(out), C.byref(n)))
        return out[: n.value]

    def mapping_digest(self, s: Setup) -> int:
        c = self.ctx(s)
        d = C.c_uint64()
        self._check(self.lib.umcref_mapping_digest(c.h, C.byref(d)))
        return d.value

    def serialize_mapping(self, s: Setup) -> bytes:
        c = self.ctx(s)
        p, n = u8p(), C.c_uint64()
        self._check(self.lib.umcref_serialize_mapping(c.h, C.byref(p), C.byref(n)))
        return _bytes_out(self, p, n)

    # -- codec ----------------------------------------------------------------
    def encode(self, v, predictor=1, dims=None, tau=1e-3, codec_id=0, backend_id=0) -> bytes:
        v = np.ascontiguousarray(v, np.float64)
        dims = np.array(dims if dims is not None else [len(v)], np.uint64)
        p, n = u8p(), C.c_uint64()
        self._check(self.lib.umcref_encode(_ptr(v, f64p), len(v), predictor, len(dims),
                                           _ptr(dims, u64p), tau, codec_id, backend_id,
                                           C.byref(p), C.byref(n)))
        return _bytes_out(self, p, n)

    def baseline_archive(self, x, name="x", tau=1e-3, rho=0.5, bound_kind=1, codec_id=0) -> bytes:
        x = np.ascontiguousarray(x, np.float64)
        p, n = u8p(), C.c_uint64()
        self._check(self.lib.umcref_baseline_archive(_ptr(x, f64p), len(x), name.encode(), C.c_double(tau),
                                                     C.c_double(rho), bound_kind, codec_id, C.byref(p),
                                                     C.byref(n)))
        return _bytes_out(self, p, n)

    def decode(self, payload: bytes, n_cap: int) -> np.ndarray:
        buf = np.frombuffer(payload, np.uint8)
        out = np.empty(max(n_cap, 1), np.float64)
        n = C.c_uint64()
        self._check(self.lib.umcref_decode(_ptr(buf, u8p), len(buf), _ptr(out, f64p), len(out),
                                           C.byref(n)))
        return out[: n.value]

    def rle_compress(self, data: bytes) -> bytes:
        buf = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
        p, n = u8p(), C.c_uint64()
        self._check(self.lib.umcref_rle_compress(_ptr(buf, u8p), len(data), C.byref(p), C.byref(n)))
        return _bytes_out(self, p, n)

    def rle_decompress(self, data: bytes) -> bytes:
        buf = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
        p, n = u8p(), C.c_uint64()
        self._check(self.lib.umcref_rle_decompress(_ptr(buf, u8p), len(data), C.byref(p), C.byref(n)))
        return _bytes_out(self, p, n)

    def split_budget(self, tau_abs, rho, coeff_abs_sum=1.0):
        a, b = C.c_double(), C.c_double()
        self._check(self.lib.umcref_split_budget(tau_abs, rho, coeff_abs_sum, C.byref(a), C.byref(b)))
        return a.value, b.value

    # -- static inputs --------------------------------------------------------
    def grid_init(self, coords, cells=None, arity=3, percentile_k=50.0, g_max=4096, delta=5.0, thr=0.35):
        coords = np.ascontiguousarray(coords, np.float64)
        n_v, dim = coords.shape
        cl = np.ascontiguousarray(cells, np.uint64) if cells is not None else np.zeros(1, np.uint64)
        n_c = len(cells) if cells is not None else 0
        osz = np.zeros(dim, np.uint64)
        oax = f64p()
        self._check(self.lib.umcref_grid_init(dim, n_v, _ptr(coords, f64p), arity, n_c, _ptr(cl, u64p),
                                              C.c_double(percentile_k), C.c_uint64(g_max), C.c_double(delta),
                                              C.c_double(thr), _ptr(osz, u64p), C.byref(oax)))
        tot = int(osz.sum())
        cat = np.ctypeslib.as_array(oax, (max(tot, 1),))[:tot].copy()
        self.lib.umcref_free(oax)
        out, off = [], 0
        for d in range(dim):
            out.append(cat[off: off + int(osz[d])])
            off += int(osz[d])
        return out

    def grid_coarsen(self, dim, coords, axes, seed_threshold=0.35):
        coords = np.ascontiguousarray(coords, np.float64)
        n_v = coords.shape[0]
        sizes = np.array([len(a) for a in axes], np.uint64)
        cat = np.ascontiguousarray(np.concatenate(axes), np.float64)
        osz = np.zeros(dim, np.uint64)
        oax, oas, ovi = f64p(), u64p(), u64p()
        mode, nvis, frac = C.c_int(), C.c_uint64(), C.c_double()
        self._check(self.lib.umcref_grid_coarsen(dim, n_v, _ptr(coords, f64p), _ptr(sizes, u64p),
                                                 _ptr(cat, f64p), seed_threshold, _ptr(osz, u64p),
                                                 C.byref(oax), C.byref(mode), C.byref(oas),
                                                 C.byref(nvis), C.byref(ovi), C.byref(frac)))
        return self._setup_from(dim, osz, oax, mode, n_v, oas, nvis, ovi, coords), frac.value

    def _setup_from(self, dim, osz, oax, mode, n_v, oas, nvis, ovi, coords):
        tot = int(osz.sum())
        cat = np.ctypeslib.as_array(oax, (tot,)).copy()
        axes, off = [], 0
        for d in range(dim):
            axes.append(cat[off: off + int(osz[d])].copy())
            off += int(osz[d])
        assign = np.ctypeslib.as_array(oas, (max(n_v, 1),))[:n_v].copy()
        vis = np.ctypeslib.as_array(ovi, (max(nvis.value, 1),))[: nvis.value].copy()
        for p in (oax, oas, ovi):
            self.free(p)
        return Setup(dim=dim, axes=axes, mode=mode.value, assignments=assign, visited=vis,
                     coords=coords)

    def build_case(self, dim, n_target, mesh_style=0, field_kind=0, seed=0):
        """gen_mesh -> gen_field -> grid_init -> grid_coarsen, as the reference tests do."""
        n_v = C.c_uint64()
        cp, vp, oax, oas, ovi = f64p(), f64p(), f64p(), u64p(), u64p()
        osz = np.zeros(dim, np.uint64)
        mode, nvis = C.c_int(), C.c_uint64()
        self._check(self.lib.umcref_build_case(dim, n_target, mesh_style, field_kind, seed,
                                               C.byref(n_v), C.byref(cp), C.byref(vp),
                                               _ptr(osz, u64p), C.byref(oax), C.byref(mode),
                                               C.byref(oas), C.byref(nvis), C.byref(ovi)))
        n = n_v.value
        coords = np.ctypeslib.as_array(cp, (n * dim,)).reshape(n, dim).copy()
        values = np.ctypeslib.as_array(vp, (n,)).copy()
        self.free(cp)
        self.free(vp)
        return self._setup_from(dim, osz, oax, mode, n, oas, nvis, ovi, coords), values

    def make_golden(self, seed=7):
        g, m, a = u8p(), u8p(), u8p()
        gl, ml, al = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._check(self.lib.umcref_make_golden(seed, C.byref(g), C.byref(gl), C.byref(m),
                                                C.byref(ml), C.byref(a), C.byref(al)))
        return _bytes_out(self, g, gl), _bytes_out(self, m, ml), _bytes_out(self, a, al)


class _Ctx:
    def __init__(self, ref, h):
        self.ref, self.h = ref, h

    def __del__(self):
        try:
            self.ref.lib.umcref_ctx_destroy(self.h)
        except Exception:
            pass


class Oracle:
    """The plain-C restatement (oracle/liboracle.so)."""

    def __init__(self, path: str = ORACLE_SO):
        self.lib = L = C.CDLL(path)
        L.umco_last_error.restype = C.c_char_p
        L.umco_free.argtypes = [C.c_void_p]
        L.umco_fnv1a64.restype = C.c_uint64
        L.umco_fnv1a64.argtypes = [u8p, C.c_uint64, C.c_uint64]
        L.umco_rle_compress.argtypes = [u8p, C.c_uint64, C.POINTER(u8p), u64p]
        L.umco_rle_decompress.argtypes = [u8p, C.c_uint64, C.POINTER(u8p), u64p]
        L.umco_encode.argtypes = [f64p, C.c_uint64, C.c_int, C.c_int, u64p, C.c_double,
                                  C.POINTER(u8p), u64p]
        L.umco_decode.argtypes = [u8p, C.c_uint64, C.POINTER(f64p), u64p]
        L.umco_split_budget.argtypes = [C.c_double, C.c_double, C.c_double, f64p, f64p]
        L.umco_mapping_digest.restype = C.c_uint64
        L.umco_mapping_digest.argtypes = [C.POINTER(_Oracle)]
        L.umco_interpolate_to_grid.argtypes = [C.POINTER(_Oracle), f64p, C.c_int, f64p]
        L.umco_residuals.argtypes = [C.POINTER(_Oracle), f64p, C.c_int, C.c_int, f64p]
        L.umco_compress.argtypes = [C.POINTER(_Oracle), f64p, C.c_char_p, C.POINTER(_OParams),
                                    C.POINTER(u8p), u64p]
        L.umco_decompress.argtypes = [C.POINTER(_Oracle), u8p, C.c_uint64, f64p]
        self.free = L.umco_free

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.umco_last_error().decode())

    def _setup(self, s: Setup):
        sizes, cat = s.axis_arrays()
        keep = [sizes, cat, np.ascontiguousarray(s.assignments, np.uint64),
                np.ascontiguousarray(s.visited, np.uint64) if len(s.visited) else np.zeros(1, np.uint64),
                None if s.coords is None else np.ascontiguousarray(s.coords, np.float64)]
        st = _Oracle(s.dim, _ptr(keep[0], u64p), _ptr(keep[1], f64p), s.mode, s.n_v,
                     _ptr(keep[2], u64p), len(s.visited), _ptr(keep[3], u64p),
                     _ptr(keep[4], f64p))
        return st, keep

    def fnv1a64(self, data: bytes, seed=0xcbf29ce484222325) -> int:
        buf = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
        return self.lib.umco_fnv1a64(_ptr(buf, u8p), len(data), seed)

    def rle_compress(self, data: bytes) -> bytes:
        buf = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
        p, n = u8p(), C.c_uint64()
        self._check(self.lib.umco_rle_compress(_ptr(buf, u8p), len(data), C.byref(p), C.byref(n)))
        return _bytes_out(self, p, n)

    def rle_decompress(self, data: bytes) -> bytes:
        buf = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
        p, n = u8p(), C.c_uint64()
        self._check(self.lib.umco_rle_decompress(_ptr(buf, u8p), len(data), C.byref(p), C.byref(n)))
        return _bytes_out(self, p, n)

    def encode(self, v, predictor=1, dims=None, tau=1e-3) -> bytes:
        v = np.ascontiguousarray(v, np.float64)
        dims = np.array(dims if dims is not None else [len(v)], np.uint64)
        p, n = u8p(), C.c_uint64()
        self._check(self.lib.umco_encode(_ptr(v, f64p), len(v), predictor, len(dims),
                                         _ptr(dims, u64p), tau, C.byref(p), C.byref(n)))
        return _bytes_out(self, p, n)

    def decode(self, payload: bytes) -> np.ndarray:
        buf = np.frombuffer(payload, np.uint8) if payload else np.zeros(1, np.uint8)
        p, n = f64p(), C.c_uint64()
        self._check(self.lib.umco_decode(_ptr(buf, u8p), len(payload), C.byref(p), C.byref(n)))
        out = np.ctypeslib.as_array(p, (max(n.value, 1),))[: n.value].copy()
        self.free(p)
        return out

    def split_budget(self, tau_abs, rho, coeff_abs_sum=1.0):
        a, b = C.c_double(), C.c_double()
        self._check(self.lib.umco_split_budget(tau_abs, rho, coeff_abs_sum, C.byref(a), C.byref(b)))
        return a.value, b.value

    def mapping_digest(self, s: Setup) -> int:
        st, keep = self._setup(s)
        return self.lib.umco_mapping_digest(C.byref(st))

    def interpolate_to_grid(self, s: Setup, x, fill=0) -> np.ndarray:
        st, keep = self._setup(s)
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(max(s.n1, 1), np.float64)
        self._check(self.lib.umco_interpolate_to_grid(C.byref(st), _ptr(x, f64p), fill,
                                                      _ptr(out, f64p)))
        return out[: s.n1]

    def residuals(self, s: Setup, x, fill=0, g_kind=0) -> np.ndarray:
        st, keep = self._setup(s)
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(max(s.n_v, 1), np.float64)
        self._check(self.lib.umco_residuals(C.byref(st), _ptr(x, f64p), fill, g_kind, _ptr(out, f64p)))
        return out[: s.n_v]

    def compress(self, s: Setup, x, name="x", tau=1e-3, rho=0.5, bound_kind=1, g_kind=0,
                 coeff_abs_sum=1.0, fill=0) -> bytes:
        st, keep = self._setup(s)
        x = np.ascontiguousarray(x, np.float64)
        prm = _OParams(tau, rho, coeff_abs_sum, bound_kind, g_kind, fill)
        p, n = u8p(), C.c_uint64()
        self._check(self.lib.umco_compress(C.byref(st), _ptr(x, f64p), name.encode(), C.byref(prm),
                                           C.byref(p), C.byref(n)))
        return _bytes_out(self, p, n)

    def decompress(self, s: Setup, archive: bytes) -> np.ndarray:
        st, keep = self._setup(s)
        buf = np.frombuffer(archive, np.uint8) if archive else np.zeros(1, np.uint8)
        out = np.empty(max(s.n_v, 1), np.float64)
        self._check(self.lib.umco_decompress(C.byref(st), _ptr(buf, u8p), len(archive),
                                             _ptr(out, f64p)))
        return out[: s.n_v]


class HostGen:
    """Host generator of the BASELINE synthetic inputs (oracle/datagen_host.c):
    the same bytes as umcg_gen_config, without the product library."""

    def __init__(self, path: str = DATAGEN_SO, threads: int | None = None):
        self.lib = L = C.CDLL(path)
        L.dgh_gen.argtypes = [C.c_int, C.c_uint64, C.c_uint64, f64p, C.c_void_p, u64p, C.c_int]
        L.dgh_gen3_block.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p, f64p, f64p, u64p, C.c_int]
        self.threads = threads or (os.cpu_count() or 1)

    def gen(self, config: int, lattice: int, seed: int, coords=True, values=True):
        n = C.c_uint64()
        if self.lib.dgh_gen(config, lattice, seed, None, None, C.byref(n), 1):
            raise ValueError("bad config / lattice")
        n = n.value
        dim = 3 if config in (3, 5) else 2
        xyz = np.empty((n, dim), np.float64) if coords else None
        vals = (np.empty((5, n), np.float32) if config == 4 else np.empty(n, np.float64)) if values else None
        rc = self.lib.dgh_gen(config, lattice, seed, _ptr(xyz, f64p),
                              None if vals is None else vals.ctypes.data_as(C.c_void_p), C.byref(C.c_uint64()),
                              self.threads)
        if rc:
            raise RuntimeError(f"dgh_gen failed ({rc})")
        return xyz, vals

    def gen3_block(self, lattice: int, seed: int, lo, hi, coords=True, values=True):
        """Config 3 restricted to lattice points in [lo, hi) per axis, in the
        full mesh's (permuted) vertex order."""
        lo = np.ascontiguousarray(lo, np.uint64)
        hi = np.ascontiguousarray(hi, np.uint64)
        n = int(np.prod(hi.astype(np.int64) - lo.astype(np.int64)))
        xyz = np.empty((n, 3), np.float64) if coords else None
        vals = np.empty(n, np.float64) if values else None
        cnt = C.c_uint64()
        rc = self.lib.dgh_gen3_block(lattice, seed, _ptr(lo, u64p), _ptr(hi, u64p), _ptr(xyz, f64p),
                                     _ptr(vals, f64p), C.byref(cnt), self.threads)
        if rc or cnt.value != n:
            raise RuntimeError(f"dgh_gen3_block failed ({rc})")
        return xyz, vals
