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


def test_bench_gpus_n_self_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks (torch.distributed.run on
    127.0.0.1); --dry-run runs the rank plumbing on CPU/gloo. The single JSON line comes from rank 0
    and its n_gpus equals the ranks that actually ran."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run", "--steps", "1", "--warmup", "3"],
                       cwd=root, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["ranks_ran"] == 2 and d["value"] > 0


def test_bench_rejects_world_size_mismatch():
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--dry-run", "--steps", "1"], cwd=root,
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode == 2 and "WORLD_SIZE" in json.loads(r.stdout.strip().splitlines()[-1])["error"]
