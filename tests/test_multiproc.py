"""Multi-process host logic of bench.py on CPU (gloo, world size 2): the
bundle stream is sharded contiguously with no overlap and no gap, and the
per-rank times reduce with MAX (the multi-GPU timing rule)."""
import os
import socket
import subprocess
import sys

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


def _plan_lib():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2112_00821_b200 import Backend
    return Backend(os.path.join(ROOT, "paper_2112_00821_b200", "_lib", "libfmvs.so"), "fmvs_",
                   needs_context=False)


def _window(i, m, ws):
    st = min(max(i - ws // 2, 0), m - ws)
    return range(st, st + ws)


@pytest.mark.parametrize("m,shards", [(512, 8), (9, 2), (7, 3), (3, 3), (20, 6), (6, 1), (11, 11)])
def test_sequence_plan_covers_windows(m, shards):
    """fmvs_sequence_plan (the multi-GPU sequence driver's shard / halo plan):
    contiguous shards; a shard imports exactly the geometric-window members
    (tools/fassmvs.cpp:163-172) it does not own, and each import is exported
    by its owner."""
    lib = _plan_lib()
    ws = min(5, m)
    plans = [lib.sequence_plan(m, shards, s, ws) for s in range(shards)]
    assert [i for p in plans for i in range(p["begin"], p["end"])] == list(range(m))
    owner = {i: s for s, p in enumerate(plans) for i in range(p["begin"], p["end"])}
    for s, p in enumerate(plans):
        need = sorted({k for i in range(p["begin"], p["end"]) for k in _window(i, m, ws) if owner[k] != s})
        assert p["imports"] == need
        for k in need:
            assert k in plans[owner[k]]["exports"]
    exported = {k for p in plans for k in p["exports"]}
    assert exported == {k for p in plans for k in p["imports"]}
    # no geometric filter: no halo
    assert all(not lib.sequence_plan(m, shards, s, 0)["imports"] for s in range(shards))


def _plan_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = _plan_lib()
    mine = lib.sequence_plan(512, world, rank, 5)
    plans = [None] * world
    dist.all_gather_object(plans, mine)
    q.put((rank, plans))
    dist.barrier()
    dist.destroy_process_group()


def test_sequence_halo_plan_gloo():
    """Two ranks (one per GPU in production) each plan their shard of the C5
    stream; gathered over gloo, every import of one rank is an export of the
    other (the halo that crosses NVLink), and the shards tile the stream."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, plans in res:
        assert plans[0]["end"] == plans[1]["begin"] == 256
        assert plans[0]["imports"] == plans[1]["exports"] == [256, 257]
        assert plans[1]["imports"] == plans[0]["exports"] == [254, 255]


@pytest.mark.parametrize("gpus", [3])
def test_bench_refuses_missing_gpus(gpus):
    """More GPUs requested than visible: a loud failure, never n_gpus: 1."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("FMVS_BENCH_SHARE_DEVICE", None)
    env["CUDA_VISIBLE_DEVICES"] = "0"  # at most one GPU visible
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(gpus), "--workload", "c1", "--steps", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0
    assert "GPU(s) visible" in r.stderr
