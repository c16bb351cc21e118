"""GPU: the C++ drop-in (include/umc_b200/pipeline_gpu.hpp) called at the
reference's own call shape, against the reference compiled in the same
binary (tests/cpp/test_wrapper.cpp). Every archive must be byte-identical to
the reference's, or differ only by codes in the quantizer's rounding window:
the binary dumps each differing case and helpers.check_archive classifies
every differing code (no unexplained difference is tolerated)."""
import os
import struct
import subprocess

import numpy as np
import pytest

from helpers import check_archive
from oracle.bindings import Setup

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "_build", "test_wrapper")


def _load_dump(path):
    b = open(path, "rb").read()
    magic, dim, mode, ml, fill, rel = struct.unpack_from("<6I", b, 0)
    assert magic == 0x4d434d55
    tau, rho = struct.unpack_from("<2d", b, 24)
    o = 40
    axes = []
    for _ in range(dim):
        (k,) = struct.unpack_from("<Q", b, o)
        axes.append(np.frombuffer(b, np.float64, k, o + 8).copy())
        o += 8 + 8 * k
    (n,) = struct.unpack_from("<Q", b, o)
    assign = np.frombuffer(b, np.uint64, n, o + 8).copy()
    o += 8 + 8 * n
    (nv,) = struct.unpack_from("<Q", b, o)
    visited = np.frombuffer(b, np.uint64, nv, o + 8).copy()
    o += 8 + 8 * nv
    x = np.frombuffer(b, np.float64, n, o).copy()
    o += 8 * n
    coords = np.frombuffer(b, np.float64, n * dim, o).copy().reshape(n, dim)
    o += 8 * n * dim
    ars = []
    for _ in range(2):
        (k,) = struct.unpack_from("<Q", b, o)
        ars.append(b[o + 8:o + 8 + k])
        o += 8 + k
    s = Setup(dim=dim, axes=axes, mode=mode, assignments=assign, visited=visited, coords=coords)
    p = dict(tau=tau, rho=rho, g_kind=ml, fill=fill, bound_kind=rel)
    return s, x, p, ars[0], ars[1]


def test_cpp_dropin_wrapper(cuda, oracle, tmp_path):
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} not built (make -C tests/cpp where /root/reference exists)")
    r = subprocess.run([BIN, str(tmp_path)], capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    last = [l for l in r.stdout.splitlines() if l.startswith("cases")][-1]
    total, exact = int(last.split()[1]), int(last.split()[3])
    dumps = sorted(tmp_path.glob("mismatch_*.bin"))
    assert total >= 16 and exact + len(dumps) == total, last
    for d in dumps:  # every differing archive: rounding-window codes only
        s, x, p, ref_ar, gpu_ar = _load_dump(d)
        check_archive(gpu_ar, ref_ar, s, x, p, oracle, d.name)
