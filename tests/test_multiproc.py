"""Multi-GPU host logic on CPU: bench.py's replica aggregation over a world-size-2 gloo group
(max over ranks for the time, sum for the work), the path `bench.py --gpus N` takes under
torchrun (replicas only, no data-path collective)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = [120.0, 95.0][rank]
    flops = [1.0e10, 2.0e10][rank]
    t, f, e = bench.reduce_over_ranks(ms, flops, 0.5 + rank, dist, "cpu")
    out[rank] = (t, f, e)
    dist.barrier()
    dist.destroy_process_group()


def test_replica_aggregation_gloo():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        for r in range(2):
            t, f, e = out[r]
            assert t == 120.0
            assert f == pytest.approx(3.0e10)
            assert e == pytest.approx(2.0)


def test_single_rank_is_identity():
    import bench
    assert bench.reduce_over_ranks(7.0, 3.0, 1.5, None, "cpu") == (7.0, 3.0, 1.5)
