"""The host generator of the synthetic inputs (oracle/datagen_host.c) against
the device generator (csrc/datagen.cu): byte-identical coordinates and fields
for every BASELINE config, so the CPU reference arm of bench.py can build
the same workload without loading the product library."""
import numpy as np
import pytest

from oracle.bindings import HostGen


def test_block_sample_is_the_full_mesh_restricted():
    g = HostGen()
    xyz, x = g.gen(3, 48, 11)
    lo, hi = np.array([8, 0, 20]), np.array([40, 24, 48])
    bxyz, bx = g.gen3_block(48, 11, lo, hi)
    idx = np.rint(xyz * 47).astype(np.int64)  # jitter < h/2: rounding recovers the lattice index
    sel = np.all((idx >= lo) & (idx < hi), axis=1)
    assert bx.size == np.prod(hi - lo)
    assert np.array_equal(bx, x[sel]) and np.array_equal(bxyz, xyz[sel])


def test_thread_count_does_not_change_bytes():
    a = HostGen(threads=1).gen(5, 50000, 3)
    b = HostGen(threads=7).gen(5, 50000, 3)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.gpu
@pytest.mark.parametrize("config,lattice", [(1, 200), (2, 70000), (3, 40), (4, 150), (5, 70000)])
def test_host_generator_matches_device(cuda, config, lattice):
    import paper_2501_06910_b200 as umcg
    seed = 0x250106910 + config
    dxyz, dvals = umcg.gen_config(config, lattice, seed, device="cuda")
    hxyz, hvals = HostGen().gen(config, lattice, seed)
    assert np.array_equal(dxyz.cpu().numpy().view(np.uint64), hxyz.view(np.uint64))
    dv = dvals.cpu().numpy()
    assert dv.dtype == hvals.dtype
    assert np.array_equal(dv.view(np.uint32 if dv.dtype == np.float32 else np.uint64),
                          hvals.view(np.uint32 if hvals.dtype == np.float32 else np.uint64))


def test_reference_library_exports_the_same_generator():
    """The CPU reference arm generates its inputs with the copy of the host
    generator compiled into oracle/_ref/libumcref.so (that process loads
    nothing else from the repo): same bytes as the standalone library."""
    import os
    from oracle.bindings import REF_SO
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    a = HostGen(path=REF_SO).gen3_block(64, 9, [0, 0, 0], [32, 32, 32])
    b = HostGen().gen3_block(64, 9, [0, 0, 0], [32, 32, 32])
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
