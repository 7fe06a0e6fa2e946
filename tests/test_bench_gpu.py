"""The bench.py contract on a real GPU: one JSON line with the required keys
(metric/value/unit/e2e/roofline/clocks/gpu_launches), and the N>1 code path
(torchrun, contiguous shards, barrier + max over ranks) exercised on one GPU
by running two ranks on cuda:0 over gloo (FMVS_BENCH_SHARE_DEVICE=1, a test
hook that is never used for reported numbers)."""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

KEYS = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "clocks",
        "roofline"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def test_bench_single_gpu_contract():
    r = subprocess.run([sys.executable, "bench.py", "--workload", "c1", "--steps", "3", "--warmup", "3",
                        "--ring", "4", "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["roofline"]["peak"] > 0 and 0 <= d["roofline"]["frac"] < 1


def test_bench_self_spawns_ranks():
    """`python bench.py --gpus 2` with no launcher starts one rank per GPU
    itself (here: two ranks sharing cuda:0 through the test hook)."""
    env = dict(os.environ, FMVS_BENCH_SHARE_DEVICE="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--workload", "c1", "--steps", "3",
                        "--warmup", "3", "--ring", "4"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0


def test_bench_two_ranks_shared_device():
    env = dict(os.environ, FMVS_BENCH_SHARE_DEVICE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
                        "2", "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py",
                        "--gpus", "2", "--workload", "c1", "--steps", "3", "--warmup", "3", "--ring", "4"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"

