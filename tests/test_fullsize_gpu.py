"""Parity at the BASELINE configs' real sizes (BASELINE.json configs, SURVEY.md
§8d): the exact bench.py workloads (C1 640x480; C2 / C2-NCC / C2-PG and C3 at
1920x1080; C4 at 3840x2160, which runs the per-level compact cost-volume
arenas) through the B200 library and through the oracle (the unmodified
reference, oracle/_ref) on identical rendered frames, compared bit for bit.

Paths that only exist at scale are exercised here: the dense 128/256-plane
coarsest levels with gridDim.z plane slicing, the 511/1021-plane global
stacks of the refined levels, row offsets near 2^20 entries, compact arenas
with their host synchronisation (4K), and the certified census/NCC bounds
over millions of tiles. Also: the device renderer at full size (it produces
bench.py's inputs), the level-0 stage capture (costs, aggregate, winners,
pre-median depth) at C2, and the output digest bench.py prints for one of
its timed bundles.
"""
import json
import subprocess
import sys

import numpy as np
import pytest

import bench
from conftest import ROOT
from test_parity_gpu import assert_same

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

PKG = __import__("paper_2112_00821_b200")


def _frames(backend, name, n_frames=None):
    scene = bench.WORKLOADS[name][0]
    views = scene.get("views", 5)
    return backend.render_plane_scene(
        scene["kind"], scene["width"], scene["height"], scene["focal"], scene["depth"],
        n_frames or views, scene["step"], seed=1, tilt_deg=scene["tilt"],
        texture_scale=scene["texture"])


def _config(name):
    return bench.make_config(PKG, **bench.WORKLOADS[name][1])


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_render_fullsize(b200, oracle, name):
    """The device renderer (bench.py's input generator) at the workload size."""
    a, ga, na = _frames(b200, name)
    b, gb, nb = _frames(oracle, name)
    for va, vb in zip(a, b):
        assert va.intrinsics == vb.intrinsics
        assert_same(va.image, vb.image, "image")
    assert_same(ga, gb, "gt depth")
    assert_same(na, nb, "gt normals")


@pytest.mark.parametrize("name", ["c1", "c2", "c2ncc", "c2pg", "c3", "c4"])
def test_estimate_bundle_fullsize(b200, oracle, name):
    bundle, gt_all, _ = _frames(oracle, name)
    gt = gt_all[len(bundle) // 2]
    cfg = _config(name)
    a = b200.estimate_bundle(bundle, cfg)
    stats = b200.level_stats()
    b = oracle.estimate_bundle(bundle, cfg)
    assert_same(a.depth, b.depth, "depth")
    assert_same(a.normals, b.normals, "normals")
    assert_same(a.confidence, b.confidence, "confidence")
    h, w = bundle[0].image.shape
    assert stats[0]["width"] == w and stats[0]["height"] == h
    assert (b.depth > 0).mean() > 0.9
    # the depth is right, not just identical: median relative error to the
    # rendered ground truth below 1 % on valid pixels
    m = (b.depth > 0) & (gt > 0)
    assert np.median(np.abs(b.depth[m] - gt[m]) / gt[m]) < 0.01


def test_stage_capture_c2_level0(b200, oracle):
    """C2 level 0 stage by stage: the ragged layout (first/count/offset), the
    u16 costs, the u32 SGM aggregate, the WTA winners and the pre-median
    depth of the B200 estimate_bundle, against the oracle's staged
    restatement of pipeline.cpp:200-309 (whose final maps are asserted equal
    to the reference's estimate_bundle inside the oracle)."""
    bundle, _, _ = _frames(oracle, "c2")
    cfg = _config("c2")
    got = b200.estimate_bundle_captured(bundle, cfg, level=0)
    want = oracle.estimate_bundle_captured(bundle, cfg, level=0)
    for key in ("first", "count", "offset", "costs", "aggregate", "winners", "depth_raw"):
        assert_same(got[key], want[key], key)
    assert len(want["costs"]) > 20_000_000
    assert_same(got["result"].depth, want["result"].depth, "depth")


def test_bench_output_digest_c2(oracle):
    """bench.py's C2 line carries the sha256 of one timed bundle's maps; the
    oracle reproduces it on the same frames."""
    ring = 6
    r = subprocess.run([sys.executable, "bench.py", "--workload", "c2", "--steps", "7", "--warmup", "3",
                        "--ring", str(ring), "--no-cpu-baseline"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)["output_digest"]
    views = bench.WORKLOADS["c2"][0].get("views", 5)
    track, _, _ = _frames(oracle, "c2", n_frames=ring + views - 1)
    bundle = track[d["bundle"]:d["bundle"] + views]
    res = oracle.estimate_bundle(bundle, _config("c2"))
    assert bench.output_digest(res.depth, res.normals, res.confidence) == d["sha256"]
