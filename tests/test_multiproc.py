"""Multi-process host logic of bench.py on CPU (gloo, world size 2): the
bundle stream is sharded contiguously with no overlap and no gap, and the
per-rank times reduce with MAX (the multi-GPU timing rule)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = list(bench.shard(512, rank, world))
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    t = bench.reduce_max(1.5 + rank, world, "cpu")
    q.put((rank, gathered, t))
    dist.barrier()
    dist.destroy_process_group()
    del torch


@pytest.mark.parametrize("world", [2])
def test_shard_and_max_reduce_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, gathered, t in res:
        flat = [i for part in gathered for i in part]
        assert flat == list(range(512))              # contiguous, no gap, no overlap
        assert all(len(part) == 256 for part in gathered)
        assert t == 1.5 + world - 1                  # MAX over ranks


def test_shard_uneven():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    parts = [list(bench.shard(10, r, 4)) for r in range(4)]
    assert [len(p) for p in parts] == [3, 3, 2, 2]
    assert [i for p in parts for i in p] == list(range(10))
