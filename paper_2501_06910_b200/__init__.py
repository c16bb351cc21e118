"""umc-b200: B200 (sm_100a) implementation of the umc multi-component
compressor's data-parallel hot path.

Python host mirror of the reference interface (umc::compress /
umc::decompress, pipeline.hpp:117-148 / 180-210; umc::encode / umc::decode,
codec.hpp:220-441) over the C ABI in include/umcg.h (libumcg.so, built
in-tree by ``paper_2501_06910_b200.build``). Device buffers are torch CUDA
tensors; PyTorch is only the allocator and stream provider here.

There is no CPU fallback: importing works without a GPU, but every compute
call goes to libumcg.so and fails loudly if the library or the device is
missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# UMCG_LIB_PATH: an alternative build of the same library (tuning variants)
LIB_PATH = os.environ.get("UMCG_LIB_PATH") or os.path.join(HERE, "libumcg.so")

# umcg_status values == reference exception types (common.hpp:19-38)
ERROR_NAMES = {
    1: "error", 2: "malformed_file", 3: "index_out_of_range", 4: "non_finite_value",
    5: "io_failure", 6: "degenerate_mesh", 7: "empty_after_filtering",
    8: "internal_inconsistency", 9: "seed_mode_unsupported", 10: "unknown_codec",
    11: "corrupt_payload", 12: "external_codec_violation", 13: "subprocess_failure",
    14: "budget_inadmissible", 15: "mapping_mismatch", 16: "zero_norm_reference",
    17: "mismatched_runs", 100: "cuda_error", 101: "invalid_argument",
}

# public symbols of include/umcg.h (checked by tests/test_abi.py)
EXPORTED = [
    "umcg_plan_create", "umcg_plan_build", "umcg_plan_destroy", "umcg_plan_clone", "umcg_plan_get_info",
    "umcg_plan_export", "umcg_compress_bound", "umcg_compress", "umcg_compress_batch",
    "umcg_decompress", "umcg_decompress_batch", "umcg_compress_host", "umcg_decompress_host",
    "umcg_decompress_host_notify", "umcg_decompress_host_parts",
    "umcg_encode_bound",
    "umcg_encode", "umcg_decode", "umcg_grid_init", "umcg_baseline_bound", "umcg_compress_baseline", "umcg_rle_bound", "umcg_rle_compress", "umcg_rle_decompress",
    "umcg_gen_config",
    "umcg_kernel_launches", "umcg_serial_fallbacks", "umcg_profile_enable", "umcg_profile_dump",
    "umcg_last_error", "umcg_version",
]


_NOTIFY = C.CFUNCTYPE(None, C.c_void_p)


class UmcgError(RuntimeError):
    """A umcg_status != 0; ``kind`` is the reference exception name."""

    def __init__(self, status: int, msg: str):
        self.status = status
        self.kind = ERROR_NAMES.get(status, str(status))
        super().__init__(f"{self.kind}: {msg}")


u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)


class GridDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("axis_sizes", u64p), ("axes", f64p)]


class MappingDesc(C.Structure):
    _fields_ = [("mode", C.c_int), ("n_vertices", C.c_uint64), ("assignments", u64p),
                ("n_visited", C.c_uint64), ("visited_nodes", u64p)]


class Params(C.Structure):
    _fields_ = [("tau", C.c_double), ("split_rho", C.c_double), ("bound_kind", C.c_int),
                ("g_kind", C.c_int), ("coeff_abs_sum", C.c_double), ("fill", C.c_int),
                ("codec_id", C.c_int), ("backend_id", C.c_int)]


class PlanInfo(C.Structure):
    _fields_ = [("dim", C.c_int), ("mode", C.c_int), ("n_vertices", C.c_uint64),
                ("n_slots", C.c_uint64), ("shape", C.c_uint64 * 3), ("n_visited", C.c_uint64),
                ("visited_fraction", C.c_double), ("digest", C.c_uint64), ("has_coords", C.c_int)]


_lib = None


def lib():
    """Load libumcg.so (raises if it was not built: no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2501_06910_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.umcg_last_error.restype = C.c_char_p
    L.umcg_version.restype = C.c_char_p
    L.umcg_kernel_launches.restype = C.c_uint64
    L.umcg_serial_fallbacks.restype = C.c_uint64
    L.umcg_profile_enable.argtypes = [C.c_int]
    L.umcg_profile_dump.restype = C.c_uint64
    L.umcg_profile_dump.argtypes = [C.c_char_p, C.c_uint64]
    L.umcg_encode_bound.restype = C.c_uint64
    L.umcg_encode_bound.argtypes = [C.c_uint64, C.c_int]
    L.umcg_grid_init.argtypes = [C.c_int, C.c_uint64, vp, C.c_int, C.c_uint64, vp, C.POINTER(GridConfig), u64p,
                                 f64p, C.c_uint64, vp]
    L.umcg_baseline_bound.restype = C.c_uint64
    L.umcg_baseline_bound.argtypes = [C.c_uint64, C.c_uint64]
    L.umcg_compress_baseline.argtypes = [C.POINTER(Params), vp, C.c_uint64, C.c_char_p, vp, C.c_uint64, u64p, vp]
    L.umcg_rle_bound.restype = C.c_uint64
    L.umcg_rle_bound.argtypes = [C.c_uint64]
    L.umcg_rle_compress.argtypes = [vp, C.c_uint64, vp, C.c_uint64, u64p, vp]
    L.umcg_rle_decompress.argtypes = [vp, C.c_uint64, vp, C.c_uint64, u64p, vp]
    L.umcg_plan_create.argtypes = [C.POINTER(GridDesc), C.POINTER(MappingDesc), C.c_int, f64p,
                                   C.POINTER(vp)]
    L.umcg_plan_build.argtypes = [C.POINTER(GridDesc), C.c_uint64, vp, C.c_double, C.c_int,
                                  C.POINTER(vp)]
    L.umcg_plan_destroy.argtypes = [vp]
    L.umcg_plan_clone.argtypes = [vp, vp]
    L.umcg_plan_get_info.argtypes = [vp, C.POINTER(PlanInfo)]
    L.umcg_plan_export.argtypes = [vp, u64p, u64p, f64p]
    L.umcg_compress_bound.argtypes = [vp, C.c_char_p, u64p]
    L.umcg_compress.argtypes = [vp, C.POINTER(Params), vp, C.c_char_p, vp, C.c_uint64, u64p, vp]
    L.umcg_compress_batch.argtypes = [vp, C.POINTER(Params), vp, C.c_int, C.c_int,
                                      C.POINTER(C.c_char_p), vp, C.c_uint64, u64p, vp]
    L.umcg_decompress.argtypes = [vp, vp, C.c_uint64, vp, vp]
    L.umcg_decompress_batch.argtypes = [vp, vp, u64p, C.c_int, C.c_int, vp, vp]
    L.umcg_decompress_host_parts.argtypes = [vp, C.POINTER(vp), u64p, C.c_int, vp]
    L.umcg_compress_host.argtypes = [vp, C.POINTER(Params), vp, C.c_char_p, vp, C.c_uint64, u64p]
    L.umcg_decompress_host.argtypes = [vp, vp, C.c_uint64, vp]
    L.umcg_decompress_host_notify.argtypes = [vp, vp, C.c_uint64, vp, vp, vp]
    L.umcg_encode.argtypes = [vp, C.c_uint64, C.c_int, C.c_int, u64p, C.c_double, C.c_int, C.c_int,
                              vp, C.c_uint64, u64p, vp]
    L.umcg_decode.argtypes = [vp, C.c_uint64, vp, C.c_uint64, u64p, vp]
    L.umcg_gen_config.argtypes = [C.c_int, C.c_uint64, C.c_uint64, vp, vp, u64p, vp]
    _lib = L
    return L


def _check(rc: int):
    if rc:
        raise UmcgError(rc, lib().umcg_last_error().decode(errors="replace"))


def kernel_launches() -> int:
    return int(lib().umcg_kernel_launches())


def serial_fallbacks() -> int:
    """Times a component used the one-thread exact replica of the reference loop."""
    return int(lib().umcg_serial_fallbacks())


def profile(enable: bool):
    """Per-kernel CUDA-event timing inside the library (hot kernels)."""
    lib().umcg_profile_enable(1 if enable else 0)


def profile_dump() -> dict:
    """{kernel: (total_ms, launches)} since the last dump."""
    buf = C.create_string_buffer(1 << 16)
    lib().umcg_profile_dump(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, ms, cnt = line.split()
        out[name] = (float(ms), int(cnt))
    return out


def _ptr(a, t):
    return a.ctypes.data_as(t)


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


@dataclass
class Budget:
    """umc::ErrorBudget (pipeline.hpp:25-29) + CompressOptions (:81-86)."""
    tau: float = 1e-3
    split_rho: float = 0.5
    bound_kind: int = 1  # 0 absolute, 1 relative_to_range
    g_kind: int = 0  # 0 nearest, 1 multilinear
    coeff_abs_sum: float = 1.0
    fill: int = 0  # 0 zero, 1 nearest_visited
    codec_id: int = 0
    backend_id: int = 0

    def c(self) -> Params:
        return Params(self.tau, self.split_rho, self.bound_kind, self.g_kind, self.coeff_abs_sum,
                      self.fill, self.codec_id, self.backend_id)


class Plan:
    """Immutable device plan for one mesh mapping (umcg_plan)."""

    def __init__(self, handle):
        self.h = handle
        info = PlanInfo()
        _check(lib().umcg_plan_get_info(self.h, C.byref(info)))
        self.info = info

    @classmethod
    def from_mapping(cls, dim, axes, mode, assignments, visited=None, coords=None):
        """umcg_plan_create: host grid + mapping (+ coordinates for multilinear g)."""
        sizes = np.array([len(a) for a in axes], np.uint64)
        cat = np.ascontiguousarray(np.concatenate([np.asarray(a, np.float64) for a in axes]))
        a = np.ascontiguousarray(assignments, np.uint64)
        v = np.ascontiguousarray(visited if visited is not None else np.zeros(0), np.uint64)
        g = GridDesc(dim, _ptr(sizes, u64p), _ptr(cat, f64p))
        m = MappingDesc(mode, len(a), _ptr(a, u64p) if len(a) else None, len(v),
                        _ptr(v, u64p) if len(v) else None)
        cp = None
        if coords is not None:
            coords = np.ascontiguousarray(coords, np.float64)
            cp = _ptr(coords, f64p)
        h = C.c_void_p()
        _check(lib().umcg_plan_create(C.byref(g), C.byref(m), dim, cp, C.byref(h)))
        return cls(h)

    @classmethod
    def build(cls, init_axes, d_coords, seed_threshold=0.35, keep_coords=False):
        """umcg_plan_build: GPU grid_coarsen of device coordinates (torch tensor [n, dim])."""
        dim = len(init_axes)
        sizes = np.array([len(a) for a in init_axes], np.uint64)
        cat = np.ascontiguousarray(np.concatenate([np.asarray(a, np.float64) for a in init_axes]))
        g = GridDesc(dim, _ptr(sizes, u64p), _ptr(cat, f64p))
        h = C.c_void_p()
        _check(lib().umcg_plan_build(C.byref(g), d_coords.shape[0], C.c_void_p(d_coords.data_ptr()),
                                     seed_threshold, 1 if keep_coords else 0, C.byref(h)))
        return cls(h)

    def clone(self) -> "Plan":
        """umcg_plan_clone: another handle on this plan with its own workspace
        (the mapping arrays are shared); calls on different handles run
        concurrently."""
        h = C.c_void_p()
        _check(lib().umcg_plan_clone(self.h, C.byref(h)))
        return Plan(h)

    def __del__(self):
        try:
            if self.h:
                lib().umcg_plan_destroy(self.h)
        except Exception:
            pass

    @property
    def n(self) -> int:
        return int(self.info.n_vertices)

    @property
    def digest(self) -> int:
        return int(self.info.digest)

    def export(self):
        """(mode, axes list, assignments u64, visited u64) back on the host."""
        n = self.n
        a = np.zeros(max(n, 1), np.uint64)
        nv = int(self.info.n_visited) if self.info.mode == 1 else 0
        v = np.zeros(max(nv, 1), np.uint64)
        shape = [int(self.info.shape[d]) for d in range(self.info.dim)]
        ax = np.zeros(sum(shape), np.float64)
        _check(lib().umcg_plan_export(self.h, _ptr(a, u64p), _ptr(v, u64p), _ptr(ax, f64p)))
        axes, off = [], 0
        for s in shape:
            axes.append(ax[off: off + s].copy())
            off += s
        return int(self.info.mode), axes, a[:n], v[:nv]

    def compress_bound(self, name: str = "") -> int:
        b = C.c_uint64()
        _check(lib().umcg_compress_bound(self.h, name.encode(), C.byref(b)))
        return b.value

    # ---- device-pointer path (the measured one) ---------------------------
    def compress_into(self, d_values, budget: Budget, d_archive, name: str = "", stream=None) -> int:
        import torch
        if d_values.dtype != torch.float64:
            raise TypeError("compress_into takes fp64 values; use compress_batch for fp32 fields")
        n = C.c_uint64()
        prm = budget.c()
        _check(lib().umcg_compress(self.h, C.byref(prm), C.c_void_p(d_values.data_ptr()),
                                   name.encode(), C.c_void_p(d_archive.data_ptr()),
                                   d_archive.numel(), C.byref(n), _stream_ptr(stream)))
        return n.value

    def decompress_into(self, d_archive, length: int, d_out, stream=None):
        _check(lib().umcg_decompress(self.h, C.c_void_p(d_archive.data_ptr()), length,
                                     C.c_void_p(d_out.data_ptr()), _stream_ptr(stream)))

    def compress(self, d_values, budget: Budget = Budget(), name: str = "") -> bytes:
        import torch
        buf = torch.empty(self.compress_bound(name), dtype=torch.uint8, device=d_values.device)
        n = self.compress_into(d_values, budget, buf, name)
        return bytes(buf[:n].cpu().numpy())

    def compress_batch_into(self, d_values, budget: Budget, d_archive, names=None, stream=None):
        """umcg_compress_batch into a device buffer: V fields [V, n] (fp64 or
        fp32, BASELINE config 4); returns the V archive lengths (archives are
        packed back to back)."""
        import torch
        V = int(d_values.shape[0])
        if d_values.dtype not in (torch.float32, torch.float64):
            raise TypeError("compress_batch takes fp32 or fp64 values")
        dtype = 1 if d_values.dtype == torch.float32 else 0
        names = names or [f"f{k}" for k in range(V)]
        lens = np.zeros(V, np.uint64)
        cn = (C.c_char_p * V)(*[nm.encode() for nm in names])
        prm = budget.c()
        _check(lib().umcg_compress_batch(self.h, C.byref(prm), C.c_void_p(d_values.data_ptr()), dtype, V, cn,
                                         C.c_void_p(d_archive.data_ptr()), d_archive.numel(), _ptr(lens, u64p),
                                         _stream_ptr(stream)))
        return lens

    def compress_batch(self, d_values, budget: Budget = Budget(), names=None) -> list:
        """umcg_compress_batch: V fields [V, n] (fp64 or fp32, BASELINE config
        4) against this plan, one archive (bytes) per field."""
        import torch
        V = int(d_values.shape[0])
        names = names or [f"f{k}" for k in range(V)]
        cap = sum(self.compress_bound(nm) for nm in names)
        buf = torch.empty(cap, dtype=torch.uint8, device=d_values.device)
        lens = self.compress_batch_into(d_values, budget, buf, names)
        host = bytes(buf[: int(lens.sum())].cpu().numpy())
        out, o = [], 0
        for ln in lens:
            out.append(host[o: o + int(ln)])
            o += int(ln)
        return out

    def decompress_batch_into(self, d_archives, lens, d_out, stream=None):
        """umcg_decompress_batch: archives packed back to back on the device
        (lens[k] bytes each, as compress_batch_into writes them) -> d_out
        [V, n] fp64 or fp32 (BASELINE config 4)."""
        import torch
        lens = np.ascontiguousarray(lens, np.uint64)
        V = int(lens.size)
        if d_out.dtype not in (torch.float32, torch.float64) or tuple(d_out.shape) != (V, self.n):
            raise TypeError("d_out must be [V, n] fp32 or fp64")
        dtype = 1 if d_out.dtype == torch.float32 else 0
        _check(lib().umcg_decompress_batch(self.h, C.c_void_p(d_archives.data_ptr()), _ptr(lens, u64p), V, dtype,
                                           C.c_void_p(d_out.data_ptr()), _stream_ptr(stream)))
        return d_out

    def decompress_batch(self, archives: list, dtype=None, device="cuda"):
        """V archives (bytes) -> [V, n] tensor (fp64 unless dtype=torch.float32)."""
        import torch
        lens = np.array([len(a) for a in archives], np.uint64)
        buf = torch.from_numpy(np.frombuffer(b"".join(archives), np.uint8).copy()).to(device)
        out = torch.empty((len(archives), self.n), dtype=dtype or torch.float64, device=device)
        return self.decompress_batch_into(buf, lens, out)

    def decompress(self, archive: bytes, device="cuda"):
        import torch
        a = torch.from_numpy(np.frombuffer(archive, np.uint8).copy()).to(device)
        out = torch.empty(self.n, dtype=torch.float64, device=device)
        self.decompress_into(a, len(archive), out)
        return out

    # ---- host-buffer path (reference call shape) ---------------------------
    def compress_host(self, values: np.ndarray, budget: Budget = Budget(), name: str = "",
                      out: np.ndarray | None = None) -> bytes | int:
        v = np.ascontiguousarray(values, np.float64)
        buf = out if out is not None else np.empty(self.compress_bound(name), np.uint8)
        n = C.c_uint64()
        prm = budget.c()
        _check(lib().umcg_compress_host(self.h, C.byref(prm), C.c_void_p(v.ctypes.data),
                                        name.encode(), C.c_void_p(buf.ctypes.data), len(buf),
                                        C.byref(n)))
        return n.value if out is not None else buf[: n.value].tobytes()

    def decompress_host(self, archive, out: np.ndarray | None = None, uploaded=None) -> np.ndarray:
        """uploaded: optional callable (umcg_decompress_host_notify), run as
        soon as the next host->device copy can be queued without delaying this
        archive's upload. It does NOT mean the archive buffer may be reused:
        a pinned mapped archive is read by the SMs during the call, so the
        buffer stays in use until this call returns."""
        a = np.frombuffer(archive, np.uint8) if isinstance(archive, (bytes, bytearray)) else archive
        length = len(archive) if isinstance(archive, (bytes, bytearray)) else int(a.size)
        y = out if out is not None else np.empty(self.n, np.float64)
        if uploaded is None:
            _check(lib().umcg_decompress_host(self.h, C.c_void_p(a.ctypes.data), length,
                                              C.c_void_p(y.ctypes.data)))
        else:
            cb = _NOTIFY(lambda _ctx: uploaded())
            _check(lib().umcg_decompress_host_notify(self.h, C.c_void_p(a.ctypes.data), length,
                                                     C.c_void_p(y.ctypes.data), C.cast(cb, C.c_void_p), None))
        return y


class HostPipeline:
    """Host-buffer round trips (compress_host -> host archive -> decompress_host)
    of a sequence of fields, overlapped across fields.

    Compress calls run on ``plans_c`` and decompress calls on ``plans_d``,
    one host thread per plan, fields dealt round-robin; all plans are handles
    on the same mesh -- ``Plan.clone()`` gives one with its own workspace and
    shared mapping arrays (archives are interchangeable: same mapping
    digest). Each host call runs on its own
    CUDA stream (api.cu host_stream), so uploads, device work and downloads
    of different fields overlap -- field uploads on one PCIe direction while
    earlier fields' outputs download on the other. Archives pass through host
    memory exactly as with sequential calls; pinned archive slots are read by
    the SMs directly (no copy-engine queueing behind a field upload).
    ``len(archive_slots)`` bounds the archives in flight
    (>= len(plans_c) + len(plans_d)).
    """

    def __init__(self, plans_c, plans_d, archive_slots):
        as_list = lambda p: list(p) if isinstance(p, (list, tuple)) else [p]  # noqa: E731
        plans_c, plans_d = as_list(plans_c), as_list(plans_d)
        every = plans_c + plans_d
        if len({id(p) for p in every}) != len(every):
            raise ValueError("HostPipeline needs distinct plans (one per worker)")
        if len(archive_slots) < len(every):
            raise ValueError("HostPipeline needs len(plans_c) + len(plans_d) archive slots")
        self.pcs, self.pds, self.slots = plans_c, plans_d, archive_slots
        self._workers = []

    def _start(self):
        import queue
        import threading

        for _ in self.pcs + self.pds:
            jobs: "queue.Queue" = queue.Queue()

            def loop(jobs=jobs):
                while True:
                    job = jobs.get()
                    if job is None:
                        return
                    job()

            t = threading.Thread(target=loop, daemon=True)
            t.start()
            self._workers.append((jobs, t))

    def run(self, fields, budget: "Budget", outs, name: str = ""):
        """Round-trip fields[k] -> outs[k] (host float64 arrays); returns the
        archive length of each field."""
        import threading

        if not self._workers:
            self._start()
        nk, Wc, Wd, S = len(fields), len(self.pcs), len(self.pds), len(self.slots)
        lens = [0] * nk
        ready = [threading.Event() for _ in range(nk)]      # archive k is in its slot
        slot_free = [threading.Event() for _ in range(nk)]  # field k's slot may be reused
        err = []

        def fail(e):
            err.append(e)
            for ev in ready + slot_free:
                ev.set()

        def compress(w):
            try:
                for k in range(w, nk, Wc):
                    if k >= S:
                        slot_free[k - S].wait()
                    if err:
                        return
                    lens[k] = self.pcs[w].compress_host(fields[k], budget, name, out=self.slots[k % S])
                    ready[k].set()
            except BaseException as e:  # surfaced on the caller's thread
                fail(e)

        def decompress(w, done):
            try:
                for k in range(w, nk, Wd):
                    ready[k].wait()
                    if err:
                        return
                    self.pds[w].decompress_host(self.slots[k % S][: lens[k]], out=outs[k])
                    slot_free[k].set()
            except BaseException as e:
                fail(e)
            finally:
                done.release()

        done = threading.Semaphore(0)
        for w in range(Wc):
            self._workers[w][0].put(lambda w=w: compress(w))
        for w in range(Wd):
            self._workers[Wc + w][0].put(lambda w=w: decompress(w, done))
        for _ in range(Wd):
            done.acquire()
        if err:
            raise err[0]
        return lens

    def close(self):
        for jobs, t in self._workers:
            jobs.put(None)
            t.join()
        self._workers = []


def encode(d_values, predictor: int = 1, dims=None, tau: float = 1e-3, codec_id: int = 0,
           backend_id: int = 0) -> bytes:
    """umc::encode (codec.hpp:220) on a device fp64 tensor; returns the payload bytes."""
    import torch
    n = d_values.numel()
    dims = np.array(dims if dims is not None else [n], np.uint64)
    cap = int(lib().umcg_encode_bound(n, len(dims)))
    buf = torch.empty(cap, dtype=torch.uint8, device=d_values.device)
    out = C.c_uint64()
    _check(lib().umcg_encode(C.c_void_p(d_values.data_ptr()), n, predictor, len(dims),
                             _ptr(dims, u64p), tau, codec_id, backend_id,
                             C.c_void_p(buf.data_ptr()), cap, C.byref(out), _stream_ptr()))
    return bytes(buf[: out.value].cpu().numpy())


def decode(payload: bytes, n_capacity: int | None = None, device="cuda"):
    """umc::decode (codec.hpp:364) of a payload; returns a device fp64 tensor."""
    import torch
    a = torch.from_numpy(np.frombuffer(payload, np.uint8).copy()).to(device) if payload else \
        torch.zeros(1, dtype=torch.uint8, device=device)
    if n_capacity is None:
        # header: n_elements at byte 12 (codec.hpp:231)
        n_capacity = int.from_bytes(payload[12:20], "little") if len(payload) >= 20 else 0
    out = torch.empty(max(n_capacity, 1), dtype=torch.float64, device=device)
    n = C.c_uint64()
    _check(lib().umcg_decode(C.c_void_p(a.data_ptr()), len(payload), C.c_void_p(out.data_ptr()),
                             n_capacity, C.byref(n), _stream_ptr()))
    return out[: n.value]


class GridConfig(C.Structure):
    _fields_ = [("percentile_k", C.c_double), ("g_max", C.c_uint64), ("delta", C.c_double),
                ("seed_mode_threshold", C.c_double)]


def grid_init(d_coords, d_cells=None, arity=3, percentile_k=50.0, g_max=4096, delta=5.0, seed_threshold=0.35):
    """umc::grid_init (grid_builder.hpp:201-282) on the device: the initial
    grid axes from the mesh's edge-length statistics (cell edges, or the
    1-NN point-cloud fallback when d_cells is None)."""
    dim = int(d_coords.shape[1])
    n_c = int(d_cells.shape[0]) if d_cells is not None else 0
    cfg = GridConfig(percentile_k, g_max, delta, seed_threshold)
    sizes = np.zeros(dim, np.uint64)
    _check(lib().umcg_grid_init(dim, d_coords.shape[0], C.c_void_p(d_coords.data_ptr()), arity, n_c,
                                C.c_void_p(d_cells.data_ptr()) if d_cells is not None else None, C.byref(cfg),
                                _ptr(sizes, u64p), None, 0, _stream_ptr()))
    cat = np.zeros(int(sizes.sum()), np.float64)
    _check(lib().umcg_grid_init(dim, d_coords.shape[0], C.c_void_p(d_coords.data_ptr()), arity, n_c,
                                C.c_void_p(d_cells.data_ptr()) if d_cells is not None else None, C.byref(cfg),
                                _ptr(sizes, u64p), _ptr(cat, f64p), len(cat), _stream_ptr()))
    out, off = [], 0
    for d in range(dim):
        out.append(cat[off: off + int(sizes[d])])
        off += int(sizes[d])
    return out


def compress_baseline(d_values, budget: "Budget", name: str = "") -> bytes:
    """umc::baseline_archive (pipeline.hpp:164-176) serialized: one lorenzo_1d
    component of the field at the full budget."""
    import torch
    n = d_values.numel()
    nb = name.encode()
    cap = int(lib().umcg_baseline_bound(n, len(nb)))
    buf = torch.empty(cap, dtype=torch.uint8, device=d_values.device)
    ln = C.c_uint64()
    _check(lib().umcg_compress_baseline(C.byref(budget.c()), C.c_void_p(d_values.data_ptr()), n, nb,
                                        C.c_void_p(buf.data_ptr()), cap, C.byref(ln), _stream_ptr()))
    return bytes(buf[: ln.value].cpu().numpy())


def rle_compress(data: bytes, device="cuda") -> bytes:
    """umc::rle_compress (lossless.hpp:24-51) of a byte string, on the device."""
    import torch
    n = len(data)
    a = torch.from_numpy(np.frombuffer(data, np.uint8).copy()).to(device) if n else \
        torch.zeros(1, dtype=torch.uint8, device=device)
    cap = int(lib().umcg_rle_bound(n))
    out = torch.empty(max(cap, 1), dtype=torch.uint8, device=device)
    ln = C.c_uint64()
    _check(lib().umcg_rle_compress(C.c_void_p(a.data_ptr()), n, C.c_void_p(out.data_ptr()), cap,
                                   C.byref(ln), _stream_ptr()))
    return bytes(out[: ln.value].cpu().numpy())


def rle_decompress(stream: bytes, capacity: int, device="cuda") -> bytes:
    """umc::rle_decompress (lossless.hpp:53-70) of a token stream, on the device."""
    import torch
    a = torch.from_numpy(np.frombuffer(stream, np.uint8).copy()).to(device) if stream else \
        torch.zeros(1, dtype=torch.uint8, device=device)
    out = torch.empty(max(capacity, 1), dtype=torch.uint8, device=device)
    ln = C.c_uint64()
    _check(lib().umcg_rle_decompress(C.c_void_p(a.data_ptr()), len(stream), C.c_void_p(out.data_ptr()),
                                     capacity, C.byref(ln), _stream_ptr()))
    return bytes(out[: ln.value].cpu().numpy())


def gen_config(config: int, lattice: int, seed: int, coords: bool = True, values: bool = True,
               device="cuda"):
    """Synthetic BASELINE inputs on the device: (coords [n,dim] f64, values)."""
    import torch
    n = C.c_uint64()
    _check(lib().umcg_gen_config(config, lattice, seed, None, None, C.byref(n), None))
    n = n.value
    dim = 3 if config in (3, 5) else 2
    xyz = torch.empty((n, dim), dtype=torch.float64, device=device) if coords else None
    if config == 4:
        vals = torch.empty((5, n), dtype=torch.float32, device=device) if values else None
    else:
        vals = torch.empty(n, dtype=torch.float64, device=device) if values else None
    _check(lib().umcg_gen_config(config, lattice, seed,
                                 C.c_void_p(xyz.data_ptr()) if xyz is not None else None,
                                 C.c_void_p(vals.data_ptr()) if vals is not None else None,
                                 C.byref(C.c_uint64()), _stream_ptr()))
    return xyz, vals
