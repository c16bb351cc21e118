"""Multi-process host logic of bench.py's replica mode (multi-GPU
is replicas only): rank discovery, max-over-ranks timing and the whole-job
value, on CPU with gloo, world_size 2."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(ws), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        w, r, lr = bench.dist_env()
        local_ms = 2.0 + 3.0 * rank  # rank 1 is the slow one
        ms = bench.max_over_ranks(local_ms)
        out[rank] = (w, r, lr, ms, bench.replica_value(w, 1000, ms))
    finally:
        dist.destroy_process_group()


def test_replicas_take_max_over_ranks_and_aggregate_work():
    ws, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
    assert sorted(out.keys()) == [0, 1]
    for rank in range(ws):
        w, r, lr, ms, value = out[rank]
        assert (w, r, lr) == (ws, rank, rank)
        assert ms == pytest.approx(5.0)  # max over ranks, identical on every rank
        assert value == pytest.approx(2 * 1000 * 8 / 5e-3 / 1e9)


def test_single_process_is_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(3.25) == 3.25
    assert bench.replica_value(1, 134217728, 4.0) == pytest.approx(134217728 * 8 / 4e-3 / 1e9)
