"""The 3-D grid decode of the fast decompress (DEC_Q32 codes -> per-plane 2-D
prefix -> outer scan, decode.cu k_nd3_plane / k_nd3_outer) on rectangular
grids whose sizes do not divide its tiles (32 rows / planes, 8-column lanes),
and its exactness guard: a plane whose sum of |q| reaches 2^31 fails the
verdict and the step-by-step decode runs. Reference: the inverse Lorenzo
of codec.hpp:61-80 / 426-437 through umc::decompress (pipeline.hpp:180-210)."""
import numpy as np
import pytest

import paper_2501_06910_b200 as umcg
from helpers import check_archive, check_decode
from oracle.bindings import Setup

pytestmark = pytest.mark.gpu


def _run(ref, oracle, shape, tau, kind, seed):
    import torch
    rng = np.random.default_rng(seed)
    # two jittered vertices per grid node: every node visited (dense mode)
    idx = np.stack(np.meshgrid(*[np.arange(m) for m in shape], indexing="ij"), -1).reshape(-1, 3)
    idx = np.concatenate([idx, idx])
    xyz = (idx + rng.uniform(-0.2, 0.2, idx.shape)) / np.maximum(np.array(shape) - 1, 1)
    xyz = xyz[rng.permutation(len(xyz))]
    x = np.sin(5 * xyz[:, 0]) * np.cos(3 * xyz[:, 1]) + xyz[:, 2]
    if kind == "noise":
        x = x + rng.normal(0, 1.0, len(x))
    axes = [np.linspace(xyz[:, d].min(), xyz[:, d].max(), shape[d]) for d in range(3)]
    plan = umcg.Plan.build(axes, torch.from_numpy(np.ascontiguousarray(xyz)).cuda())
    mode, gaxes, assign, visited = plan.export()
    assert mode == 0 and tuple(len(a) for a in gaxes) == tuple(shape)  # dense, grid kept as given
    s = Setup(dim=3, axes=gaxes, mode=mode, assignments=assign, visited=visited, coords=None)
    p = dict(tau=tau, rho=0.5, bound_kind=1)
    label = f"shape {shape} tau {tau} {kind}"
    got = plan.compress(torch.from_numpy(x).cuda(), umcg.Budget(tau=tau), name="f")
    want = ref.compress(s, x, name="f", tau=tau)
    check_archive(got, want, s, x, p, oracle, label)
    fb0 = umcg.serial_fallbacks()
    out = plan.decompress(got).cpu().numpy()
    check_decode(out, ref.decompress(s, got), x, tau * np.ptp(x), label)
    assert umcg.serial_fallbacks() == fb0, label


@pytest.mark.parametrize("shape", [(5, 37, 256), (70, 3, 13), (33, 65, 200), (2, 2, 1), (40, 31, 255),
                                   (1, 129, 9)])
def test_nd3_rectangular_grids_match_reference(cuda, ref, oracle, shape):
    _run(ref, oracle, shape, 1e-4, "smooth", 7)


def test_nd3_plane_guard_falls_back_exactly(cuda, ref, oracle):
    # relative tau 5e-9 on a noisy field: grid codes ~1e8, so a 13 x 13 plane
    # sums |q| past 2^31 -- the int32 plane prefix is not trusted and the
    # step-by-step decode (int64 prefix) must give the reference's values
    _run(ref, oracle, (6, 13, 13), 5e-9, "noise", 11)
