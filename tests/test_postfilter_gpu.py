"""Parity of the post-filters and the sequence driver
against the oracle: dog_mask / apply_mask / geometric_consistency_mask
(postfilter.cpp) and the `fassmvs estimate` loop (tools/fassmvs.cpp:92-176)
restated over the reference library (oracle/ref_capi.cpp,
ref_estimate_sequence). All outputs are compared bit for bit. The cases
follow the reference's own test_postfilter.cpp: flat images, a dense
checkerboard, a checkerboard with a flat patch (the morphology replay case),
rendered scenes, identical / corrupted / disjoint windows, both depth
lookups, and the configuration errors."""
import numpy as np
import pytest

from paper_2112_00821_b200 import (ConfigError, ConsistencyView, DepthLookup, Filter,
                                   GeomFilterConfig, InvalidInputError, SgmVariant)

from scenes import config, render

pytestmark = pytest.mark.gpu


def assert_same(a, b, what):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, what
    if not np.array_equal(a, b, equal_nan=True):
        bad = np.argwhere(a != b)
        raise AssertionError(f"{what}: {len(bad)} mismatches, first at {bad[:5].tolist()}")


def checkerboard(w, h, cell):
    y, x = np.mgrid[0:h, 0:w]
    return np.where(((x // cell + y // cell) & 1) == 1, 220, 40).astype(np.uint8)


def _images(rng):
    cb = checkerboard(96, 80, 4)
    patch = cb.copy()
    patch[20:60, 28:68] = 128  # test_postfilter.cpp:80-86
    blobs = (rng.random((70, 90)) < 0.08).astype(np.uint8) * 200 + 20
    quant = ((rng.random((64, 64)) * 4).astype(np.uint8) * 60)
    gentle = (np.add.outer(np.arange(50), np.arange(75)) // 7 * 3 % 256).astype(np.uint8)
    return {"constant": np.full((36, 48), 120, np.uint8), "checker": checkerboard(64, 48, 4),
            "checker_patch": patch, "blobs": blobs, "quantized": quant, "gentle": gentle,
            "noise": rng.integers(0, 256, (61, 83)).astype(np.uint8),
            "tiny": np.array([[3, 200], [10, 7]], np.uint8), "row": rng.integers(0, 256, (1, 40)).astype(np.uint8)}


@pytest.mark.parametrize("name", ["constant", "checker", "checker_patch", "blobs", "quantized",
                                  "gentle", "noise", "tiny", "row", "rendered"])
def test_dog_mask_bitexact(b200, oracle, rng, name):
    if name == "rendered":
        bundle, _, _ = render(oracle, "slanted", 160, 120, tilt=30.0, texture=0.35)
        img = bundle[2].image
    else:
        img = _images(rng)[name]
    a = b200.dog_mask(img)
    b = oracle.dog_mask(img)
    assert_same(a, b, f"dog_mask[{name}]")
    if name == "constant":
        assert not b.any()  # test_postfilter.cpp:66-71


def test_apply_mask_bitexact(b200, oracle, rng):
    h, w = 23, 31
    d = rng.uniform(1, 9, (h, w)).astype(np.float32)
    n = rng.normal(size=(h, w, 3)).astype(np.float32)
    c = rng.uniform(0, 1, (h, w)).astype(np.float32)
    m = (rng.random((h, w)) < 0.6).astype(np.uint8)
    a = b200.apply_mask(d, n, c, m)
    b = oracle.apply_mask(d, n, c, m)
    assert_same(a.depth, b.depth, "depth")
    assert_same(a.normals, b.normals, "normals")
    assert_same(a.confidence, b.confidence, "confidence")
    with pytest.raises(InvalidInputError):
        b200.apply_mask(d, n, c, m[:, :-1])


def _window(oracle, rng, corrupt, kind="slanted", views=5, w=96, h=72, tilt=25.0):
    bundle, gd, _ = render(oracle, kind, w, h, focal=float(w), tilt=tilt, views=views, step=0.4)
    win = []
    for k in range(views):
        d = gd[k].copy()
        if corrupt:
            bad = rng.random(d.shape) < 0.15
            d[bad] *= rng.uniform(0.5, 1.8, bad.sum()).astype(np.float32)
            d[rng.random(d.shape) < 0.05] = 0.0
            d[5:9, 10:30] = np.nan if k == 0 else d[5:9, 10:30]
        win.append(ConsistencyView(d.astype(np.float32), bundle[k].intrinsics, bundle[k].pose))
    return win


@pytest.mark.parametrize("lookup", [DepthLookup.Nearest, DepthLookup.Bilinear])
@pytest.mark.parametrize("corrupt", [False, True])
@pytest.mark.parametrize("ref_index,eta_r,eta_h", [(2, 10.0, 3), (0, 0.75, 2), (4, 0.02, 4)])
def test_geometric_consistency_bitexact(b200, oracle, rng, lookup, corrupt, ref_index, eta_r, eta_h):
    win = _window(oracle, rng, corrupt)
    cfg = GeomFilterConfig(eta_r, eta_h, lookup)
    a = b200.geometric_consistency_mask(win, ref_index, cfg)
    b = oracle.geometric_consistency_mask(win, ref_index, cfg)
    assert_same(a, b, "keep")
    if corrupt:
        assert (b == 0).any() and (b == 1).any()


def test_geometric_consistency_disjoint_and_errors(b200, oracle, rng):
    win = _window(oracle, rng, False)
    # neighbours looking at a disjoint scene (test_postfilter.cpp:221-236)
    for v in win[1:]:
        v.pose.center = np.asarray(v.pose.center, np.float64) + np.array([0.0, 0.0, -60.0])
    assert_same(b200.geometric_consistency_mask(win, 0), oracle.geometric_consistency_mask(win, 0),
                "disjoint")
    for be in (b200, oracle):
        with pytest.raises(ConfigError):
            be.geometric_consistency_mask(win[:3], 1, GeomFilterConfig(eta_h=3))
        with pytest.raises(ConfigError):
            be.geometric_consistency_mask(win, 1, GeomFilterConfig(eta_h=0))
        with pytest.raises(InvalidInputError):
            be.geometric_consistency_mask(win, 7)


SEQ_CFGS = [
    ("census_sn_2lvl", dict(d_min=4.0, d_max=40.0, levels=2, cost="census5", max_planes=64,
                            variant=SgmVariant.SurfaceNormal)),
    ("ncc_plane_1lvl", dict(d_min=6.0, d_max=16.0, levels=1, cost="ncc5", max_planes=48)),
]


@pytest.mark.parametrize("filt", [Filter.none, Filter.dog, Filter.geom, Filter.both])
@pytest.mark.parametrize("stride", [1, 2])
@pytest.mark.parametrize("name,cfg", SEQ_CFGS, ids=[c[0] for c in SEQ_CFGS])
def test_estimate_sequence_bitexact(b200, oracle, filt, stride, name, cfg):
    frames, _, _ = render(oracle, "slanted", 96, 64, tilt=30.0, views=11, step=0.35, texture=0.3)
    c = config(**cfg)
    a = b200.estimate_sequence(frames, c, stride, filt)
    b = oracle.estimate_sequence(frames, c, stride, filt)
    assert [r.frame for r in a] == [r.frame for r in b]
    assert len(b) >= 2
    for ra, rb in zip(a, b):
        assert_same(ra.maps.depth, rb.maps.depth, f"depth[{ra.frame}]")
        assert_same(ra.maps.normals, rb.maps.normals, f"normals[{ra.frame}]")
        assert_same(ra.maps.confidence, rb.maps.confidence, f"confidence[{ra.frame}]")


SHARDINGS = [([0, 0], 3, False), ([0, 0, 0], 1, True), ([0, 0, 0, 0, 0], 2, False)]


@pytest.mark.parametrize("filt", [Filter.none, Filter.dog, Filter.geom, Filter.both])
@pytest.mark.parametrize("devices,inflight,pinned", SHARDINGS, ids=["2x3", "3x1-pinned", "5x2"])
def test_estimate_sequence_multi_bitexact(b200, oracle, filt, devices, inflight, pinned):
    """fmvs_estimate_sequence_multi with several shards on one GPU (the
    cross-shard halo goes through the same cudaMemcpyPeerAsync path as on
    NVLink) reproduces the reference CLI loop bit for bit, including the
    geometric filter's windows that straddle shard boundaries; 5 shards of
    1-2 results make every result a halo export."""
    frames, _, _ = render(oracle, "slanted", 96, 64, tilt=30.0, views=13, step=0.35, texture=0.3)
    c = config(**SEQ_CFGS[0][1])
    a = b200.estimate_sequence_multi(frames, c, devices, 1, filt, inflight=inflight, pinned=pinned)
    b = oracle.estimate_sequence(frames, c, 1, filt)
    assert [r.frame for r in a] == [r.frame for r in b]
    for ra, rb in zip(a, b):
        assert_same(ra.maps.depth, rb.maps.depth, f"depth[{ra.frame}]")
        assert_same(ra.maps.normals, rb.maps.normals, f"normals[{ra.frame}]")
        assert_same(ra.maps.confidence, rb.maps.confidence, f"confidence[{ra.frame}]")


def test_estimate_sequence_multi_errors(b200):
    frames, _, _ = render(b200, "fronto", 48, 40, views=6, step=0.3)
    c = config(8.0, 12.0, levels=1, cost="census5", max_planes=32)
    with pytest.raises(ConfigError):
        b200.estimate_sequence_multi(frames, c, [0, 0], 0)
    with pytest.raises(InvalidInputError):
        b200.estimate_sequence_multi(frames[:4], c, [0], 1)
    with pytest.raises(ConfigError):
        b200.estimate_sequence_multi(frames, c, [0, 0], 1, Filter.geom)
    with pytest.raises(ConfigError):
        b200.estimate_sequence_multi(frames, c, [0], 1, inflight=0)


def test_estimate_sequence_errors(b200, oracle):
    frames, _, _ = render(oracle, "fronto", 48, 40, views=6, step=0.3)
    c = config(8.0, 12.0, levels=1, cost="census5", max_planes=32)
    for be in (b200, oracle):
        with pytest.raises(ConfigError):
            be.estimate_sequence(frames, c, 0)  # stride < 1
        c4 = config(8.0, 12.0, levels=1, cost="census5", max_planes=32, bundle_size=4)
        with pytest.raises(ConfigError):
            be.estimate_sequence(frames, c4, 1)  # even bundle
        with pytest.raises(InvalidInputError):
            be.estimate_sequence(frames[:4], c, 1)  # shorter than one bundle
        with pytest.raises(ConfigError):
            be.estimate_sequence(frames, c, 1, Filter.geom)  # 2 results < eta_h + 1
