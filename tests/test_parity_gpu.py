"""Stage-wise and end-to-end parity of the B200 CUDA path against the oracle
(the unmodified reference built against the Eigen shim), on identical seeded
inputs. Integer stages must be bit-exact; the float stages are designed to be
bit-exact as well (same FP64 expression trees, no FMA), and are asserted so.
"""
import os

import numpy as np
import pytest

from paper_2112_00821_b200 import (ConfigError, CostFunctionSpec, CostKind, CostVolume,
                                   GeometryError, Intrinsics, InvalidInputError, PlaneStack,
                                   RangeKind, RangePolicy, SgmConfig, SgmVariant)

from scenes import config, harmonic_stack, random_volume, render

pytestmark = pytest.mark.gpu

COSTS = ["census5", "census97", "ncc5", "ncc9"]


def assert_same(a, b, what):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, what
    if not np.array_equal(a, b, equal_nan=True):
        bad = np.argwhere(a != b)
        raise AssertionError(f"{what}: {len(bad)} mismatches, first at {bad[:5].tolist()}: "
                             f"{a[tuple(bad[0])]} vs {b[tuple(bad[0])]}")


# ------------------------------------------------------------- render ----
def test_render_matches_reference(b200, oracle):
    for kind, tilt in (("fronto", 0.0), ("slanted", 30.0)):
        a, ga, na = render(b200, kind, 96, 64, tilt=tilt)
        b, gb, nb = render(oracle, kind, 96, 64, tilt=tilt)
        for va, vb in zip(a, b):
            assert_same(va.image, vb.image, "image")
        assert_same(ga, gb, "gt depth")
        assert_same(na, nb, "gt normals")


def _scenes():
    """SyntheticScenes beyond a single unbounded plane (render.cpp:52-141):
    several planes with extents (nearest hit, misses), checkerboard texture,
    rotated cameras, oblique u axes, a plane seen edge-on, zero-size extents."""
    from paper_2112_00821_b200 import Intrinsics, Pose, ScenePlane, SyntheticScene, TextureKind
    from paper_2112_00821_b200 import lateral_trajectory

    def rot(ax, deg):
        c, s_ = np.cos(np.radians(deg)), np.sin(np.radians(deg))
        if ax == "y":
            return np.array([[c, 0, s_], [0, 1, 0], [-s_, 0, c]])
        return np.array([[1, 0, 0], [0, c, -s_], [0, s_, c]])

    k = Intrinsics(110.0, 104.0, 63.5, 41.0, 128, 83)
    boxes = [ScenePlane((0, 0, 9.0), (0, 0, -1), (1, 0, 0), 4.0, 2.5),
             ScenePlane((0.5, -0.3, 6.0), (0.2, 0.1, -1.0), (1, 1, 0), 1.5, 0.8),
             ScenePlane((-1.2, 0.6, 5.0), (0, -0.5, -1.0), (1, 0, 0.3), 0.7, 1.1),
             ScenePlane((0.0, 1.5, 7.0), (0, 1, 0), (1, 0, 0), 3.0, 3.0),  # seen edge-on / from below
             ScenePlane((2.0, 0.0, 4.0), (0, 0, -1), (0, 1, 0), 0.0, 0.5)]  # zero-width strip
    poses = lateral_trajectory(3, 0.4) + [Pose(rot("y", 7.0), np.array([0.3, -0.2, 0.5])),
                                          Pose(rot("x", -5.0) @ rot("y", -4.0), np.array([-0.6, 0.1, -1.0]))]
    yield "boxes_noise", SyntheticScene(boxes, poses, k, TextureKind.ValueNoise, 0.23, 5)
    yield "boxes_checker", SyntheticScene(boxes, poses, k, TextureKind.Checkerboard, 0.31, 1)
    yield "plane_checker", SyntheticScene([ScenePlane((0, 0, 10.0), (0, -0.5, -0.866))],
                                          lateral_trajectory(5, 0.59), Intrinsics(96.0, 96.0, 47.5, 31.5, 96, 64),
                                          TextureKind.Checkerboard, 0.1, 1)
    yield "behind", SyntheticScene([ScenePlane((0, 0, -3.0), (0, 0, 1))], lateral_trajectory(2, 1.0), k,
                                   TextureKind.ValueNoise, 0.5, 2)


@pytest.mark.parametrize("name", ["boxes_noise", "boxes_checker", "plane_checker", "behind"])
def test_render_scene_matches_reference(b200, oracle, name):
    scene = dict(_scenes())[name]
    a, ga, na = b200.render_scene(scene)
    b, gb, nb = oracle.render_scene(scene)
    for va, vb in zip(a, b):
        assert_same(va.image, vb.image, "image")
    assert_same(ga, gb, "gt depth")
    assert_same(na, nb, "gt normals")
    if name.startswith("boxes"):
        assert len(np.unique(a[0].image)) > 1 and (ga[0] == 0).any() and (ga[0] > 0).any()


def test_render_scene_errors_match(b200, oracle):
    from paper_2112_00821_b200 import Intrinsics, Pose, ScenePlane, SyntheticScene
    from paper_2112_00821_b200 import lateral_trajectory
    k = Intrinsics(50.0, 50.0, 15.5, 11.5, 32, 24)
    cases = [SyntheticScene([], lateral_trajectory(2, 0.5), k),
             SyntheticScene([ScenePlane()], [], k),
             SyntheticScene([ScenePlane()], lateral_trajectory(2, 0.5), Intrinsics(0.0, 50.0, 1, 1, 32, 24)),
             SyntheticScene([ScenePlane()], lateral_trajectory(2, 0.5), k, texture_scale=0.0),
             SyntheticScene([ScenePlane()], [Pose(), Pose(np.diag([1.0, 1.0, -1.0]))], k)]
    for scene in cases:
        errs = []
        for backend in (b200, oracle):
            try:
                backend.render_scene(scene)
                errs.append(None)
            except Exception as e:  # noqa: BLE001
                errs.append(type(e))
        assert errs[0] is not None and errs[0] == errs[1], errs


# ------------------------------------------------------------- stages ----
def test_build_pyramids(b200, oracle):
    bundle, _, _ = render(oracle, "slanted", 97, 61, tilt=20.0)
    pa = b200.build_pyramids(bundle, 4)
    pb = oracle.build_pyramids(bundle, 4)
    for la, lb in zip(pa, pb):
        for va, vb in zip(la, lb):
            assert va.intrinsics == vb.intrinsics
            assert_same(va.image, vb.image, "pyramid")


@pytest.mark.parametrize("kind", [RangeKind.Full, RangeKind.Fixed, RangeKind.SpacingMultiple])
def test_refine_range(b200, oracle, rng, kind):
    w, h = 57, 43
    prior = rng.uniform(3, 12, (h, w)).astype(np.float32)
    prior[rng.random((h, w)) < 0.1] = 0.0
    stack = PlaneStack(harmonic_stack(40, fb=200.0, disp0=15.0))
    intr = Intrinsics(60.0, 60.0, 28.0, 21.0, w, h)
    pol = RangePolicy(kind, 3.0 if kind != RangeKind.Fixed else 0.7)
    a = b200.refine_range(prior, pol, 3.2, 13.0, stack, intr)
    b = oracle.refine_range(prior, pol, 3.2, 13.0, stack, intr)
    assert_same(a[0], b[0], "lo")
    assert_same(a[1], b[1], "hi")


def _level_inputs(oracle, kind="slanted", w=80, h=60, tilt=25.0, views=5, step=0.5):
    bundle, _, _ = render(oracle, kind, w, h, tilt=tilt, views=views, step=step)
    ref = bundle[len(bundle) // 2]
    n = (0.0, 0.0, -1.0)
    dlo, dhi = oracle.bounding_distances(6.0, 16.0, n, ref.intrinsics)
    planes = oracle.plane_distances(ref.intrinsics, ref.pose, bundle[0].intrinsics, bundle[0].pose,
                                    dlo, dhi, n, 100000)
    return bundle, PlaneStack(planes, n)


@pytest.mark.parametrize("cost", COSTS)
def test_sweep_cost_volume_bitexact(b200, oracle, rng, cost):
    bundle, stack = _level_inputs(oracle)
    ref = bundle[2]
    h, w = ref.image.shape
    lo = np.full((h, w), 6.0, np.float32)
    hi = np.full((h, w), 16.0, np.float32)
    # ragged ranges around a random prior, some pixels empty
    mid = rng.uniform(6, 16, (h, w)).astype(np.float32)
    rad = rng.uniform(0.2, 2.0, (h, w)).astype(np.float32)
    sel = rng.random((h, w)) < 0.7
    lo[sel] = np.maximum(6.0, mid - rad)[sel]
    hi[sel] = np.minimum(16.0, mid + rad)[sel]
    lo[rng.random((h, w)) < 0.05] = 20.0  # empty intervals
    spec = {"census5": (CostKind.CensusHamming, 5, 5), "census97": (CostKind.CensusHamming, 9, 7),
            "ncc5": (CostKind.NccTruncated, 5, 5), "ncc9": (CostKind.NccTruncated, 9, 9)}[cost]
    cf = CostFunctionSpec(*spec)
    a = b200.sweep_cost_volume(bundle, 2, stack, lo, hi, cf)
    b = oracle.sweep_cost_volume(bundle, 2, stack, lo, hi, cf)
    assert a.per_side == b.per_side
    assert_same(a.first, b.first, "first")
    assert_same(a.count, b.count, "count")
    assert_same(a.offset, b.offset, "offset")
    assert_same(a.costs, b.costs, "costs")
    assert len(a.costs) > 1000


@pytest.mark.parametrize("texture", ["quantized", "noise", "constant", "ramp"])
@pytest.mark.parametrize("cost", ["census5", "census97", "ncc5", "ncc9"])
def test_sweep_certified_census_ties(b200, oracle, rng, texture, cost):
    """Flat / quantised / noisy / ramp images stress the certified FP32 census
    and NCC paths: exact FP64 ties, near-ties, flat windows (var_b <= 0) and
    costs on rounding boundaries must fall back to the reference walk. The
    constant image leaves every census bit undecided, overflowing the per-warp
    exact-sample list (lanes then walk serially)."""
    bundle, stack = _level_inputs(oracle, w=70, h=44)
    for v in bundle:
        if texture == "quantized":
            v.image = ((v.image // 48) * 48).astype(np.uint8)
        elif texture == "noise":
            v.image = rng.integers(0, 256, v.image.shape).astype(np.uint8)
        elif texture == "ramp":
            hh, ww = v.image.shape
            v.image = ((np.arange(ww)[None, :] * 3 + np.arange(hh)[:, None]) % 256).astype(np.uint8)
        else:
            v.image = np.full_like(v.image, 77)
    h, w = bundle[2].image.shape
    lo = np.full((h, w), 6.0, np.float32)
    hi = np.full((h, w), 16.0, np.float32)
    spec = {"census5": (CostKind.CensusHamming, 5, 5), "census97": (CostKind.CensusHamming, 9, 7),
            "ncc5": (CostKind.NccTruncated, 5, 5), "ncc9": (CostKind.NccTruncated, 9, 9)}[cost]
    cf = CostFunctionSpec(*spec)
    a = b200.sweep_cost_volume(bundle, 2, stack, lo, hi, cf)
    b = oracle.sweep_cost_volume(bundle, 2, stack, lo, hi, cf)
    assert_same(a.costs, b.costs, "costs")


@pytest.mark.parametrize("texture", ["scene", "smooth"])
@pytest.mark.parametrize("cost,w,h", [("census5", 640, 400), ("ncc5", 640, 400), ("ncc9", 320, 200)])
def test_sweep_certified_large(b200, oracle, rng, texture, cost, w, h):
    """Larger full-range volumes (millions of hypothesis-views) through the
    certified tiled sweeps: the rendered scene, and smooth low-gradient
    texture (blurred noise quantised to u8), whose many near-flat windows
    sit close to the NCC certification thresholds (var >= 1, rounding
    boundaries of the cost) and produce many exact census ties."""
    bundle, stack = _level_inputs(oracle, w=w, h=h)
    if texture == "smooth":
        k = np.exp(-0.5 * (np.arange(-6, 7) / 3.0) ** 2)
        k /= k.sum()
        for v in bundle:
            z = rng.normal(128.0, 60.0, v.image.shape)
            z = np.apply_along_axis(lambda r: np.convolve(r, k, "same"), 1, z)
            z = np.apply_along_axis(lambda c: np.convolve(c, k, "same"), 0, z)
            v.image = np.clip(np.round(z), 0, 255).astype(np.uint8)
    hh, ww = bundle[2].image.shape
    lo = np.full((hh, ww), 6.0, np.float32)
    hi = np.full((hh, ww), 16.0, np.float32)
    spec = {"census5": (CostKind.CensusHamming, 5, 5), "ncc5": (CostKind.NccTruncated, 5, 5),
            "ncc9": (CostKind.NccTruncated, 9, 9)}[cost]
    cf = CostFunctionSpec(*spec)
    a = b200.sweep_cost_volume(bundle, 2, stack, lo, hi, cf)
    b = oracle.sweep_cost_volume(bundle, 2, stack, lo, hi, cf)
    assert_same(a.costs, b.costs, "costs")
    assert len(a.costs) > 2_000_000, len(a.costs)


def test_sweep_mixed_wide_and_narrow(b200, oracle, rng):
    """Pixels with > 192 hypotheses (full-range, invalid prior) take the exact
    per-hypothesis kernel, the rest the tiled certified kernel, in one call."""
    bundle, _, _ = render(oracle, "slanted", 120, 40, focal=400.0, tilt=20.0, step=1.2)
    ref = bundle[2]
    n = (0.0, 0.0, -1.0)
    dlo, dhi = oracle.bounding_distances(4.0, 40.0, n, ref.intrinsics)
    planes = oracle.plane_distances(ref.intrinsics, ref.pose, bundle[0].intrinsics, bundle[0].pose,
                                    dlo, dhi, n, 100000)
    assert len(planes) > 192
    stack = PlaneStack(planes, n)
    h, w = ref.image.shape
    lo = np.full((h, w), 4.0, np.float32)
    hi = np.full((h, w), 40.0, np.float32)
    narrow = rng.random((h, w)) < 0.7
    mid = rng.uniform(8, 12, (h, w)).astype(np.float32)
    lo[narrow] = (mid - 0.5)[narrow]
    hi[narrow] = (mid + 0.5)[narrow]
    cf = CostFunctionSpec(CostKind.CensusHamming, 5, 5)
    a = b200.sweep_cost_volume(bundle, 2, stack, lo, hi, cf)
    b = oracle.sweep_cost_volume(bundle, 2, stack, lo, hi, cf)
    assert (b.count > 192).any() and (b.count[b.count > 0] <= 192).any()
    assert_same(a.costs, b.costs, "costs")


@pytest.mark.parametrize("views", [9, 11])
def test_sweep_many_views(b200, oracle, views):
    """9 views = the tiled kernel's maximum (8 matching), 11 = exact fallback path."""
    bundle, _, _ = render(oracle, "slanted", 48, 36, tilt=20.0, views=views, step=0.3)
    ref = bundle[views // 2]
    n = (0.0, 0.0, -1.0)
    dlo, dhi = oracle.bounding_distances(6.0, 16.0, n, ref.intrinsics)
    planes = oracle.plane_distances(ref.intrinsics, ref.pose, bundle[0].intrinsics, bundle[0].pose,
                                    dlo, dhi, n, 100000)
    stack = PlaneStack(planes, n)
    lo = np.full((36, 48), 6.0, np.float32)
    hi = np.full((36, 48), 16.0, np.float32)
    cf = CostFunctionSpec(CostKind.CensusHamming, 5, 5)
    a = b200.sweep_cost_volume(bundle, views // 2, stack, lo, hi, cf)
    b = oracle.sweep_cost_volume(bundle, views // 2, stack, lo, hi, cf)
    assert_same(a.costs, b.costs, "costs")


def test_sweep_three_views_rotated(b200, oracle, rng):
    """Non-lateral geometry: rotated matching views, non-fronto sweep normal."""
    bundle, _, _ = render(oracle, "slanted", 72, 54, tilt=35.0, views=3, step=0.8)
    from scenes import rotation
    bundle[0].pose.rotation = rotation(rng, 0.03)
    bundle[2].pose.rotation = rotation(rng, 0.03)
    n = np.array([0.0, -0.3, -1.0])
    n /= np.linalg.norm(n)
    ref = bundle[1]
    dlo, dhi = oracle.bounding_distances(5.0, 15.0, n, ref.intrinsics)
    planes = oracle.plane_distances(ref.intrinsics, ref.pose, bundle[0].intrinsics, bundle[0].pose,
                                    dlo, dhi, n, 100000)
    stack = PlaneStack(planes, tuple(n))
    h, w = ref.image.shape
    lo = np.full((h, w), 5.0, np.float32)
    hi = np.full((h, w), 15.0, np.float32)
    for cf in (CostFunctionSpec(CostKind.CensusHamming, 5, 5), CostFunctionSpec(CostKind.NccTruncated, 5, 5)):
        a = b200.sweep_cost_volume(bundle, 1, stack, lo, hi, cf)
        b = oracle.sweep_cost_volume(bundle, 1, stack, lo, hi, cf)
        assert_same(a.count, b.count, "count")
        assert_same(a.costs, b.costs, "costs")


def test_sweep_errors_match(b200, oracle):
    bundle, stack = _level_inputs(oracle, w=32, h=24)
    h, w = bundle[2].image.shape
    lo = np.full((h, w), 6.0, np.float32)
    hi = np.full((h, w), 16.0, np.float32)
    for be in (b200, oracle):
        with pytest.raises(ConfigError):
            be.sweep_cost_volume(bundle, 2, stack, lo, hi, CostFunctionSpec(CostKind.CensusHamming, 7, 7))
        with pytest.raises(InvalidInputError):
            be.sweep_cost_volume(bundle, 0, stack, lo, hi, CostFunctionSpec())
        with pytest.raises(InvalidInputError):
            be.sweep_cost_volume(bundle, 2, PlaneStack(stack.distances[::-1].copy()), lo, hi,
                                 CostFunctionSpec())


def _volume(planes, w, h, rng, ragged=True, max_cost=300):
    first, count, offset, costs = random_volume(rng, w, h, planes, ragged, max_cost)
    return CostVolume(w, h, PlaneStack(harmonic_stack(planes)), 2, first, count, offset, costs)


DIRS = [(1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, -1), (1, -1), (-1, 1)]


def _blocking(monkeypatch, gk):
    """Lane blocking of the SGM kernel: 'GxK' (G lanes per line, K hypotheses
    per lane and pass), '0' (one line per warp) or 'default' (the library's
    choice: G=4 x K=3 line kernel with 10-bit packed step records for the
    default range policy)."""
    if gk == "default":
        monkeypatch.delenv("FMVS_SGM_G", raising=False)
        monkeypatch.delenv("FMVS_SGM_K", raising=False)
        return
    g, _, k = gk.partition("x")
    monkeypatch.setenv("FMVS_SGM_G", g)
    monkeypatch.setenv("FMVS_SGM_K", k or "1")


@pytest.mark.parametrize("group", ["0", "4x3", "4x4", "8x2", "8x4", "32x1", "32x4"])
@pytest.mark.parametrize("adaptive", [False, True])
def test_aggregate_single_paths_bitexact(b200, oracle, rng, adaptive, group, monkeypatch):
    _blocking(monkeypatch, group)
    img = rng.integers(0, 256, (9, 13)).astype(np.uint8)
    intr = Intrinsics(100.0, 100.0, 6.0, 4.0, 13, 9)
    cfg = SgmConfig(SgmVariant.Plane, 8, 7.0, adaptive, 40.0, 8.0, 10.0, 2)
    for _ in range(4):
        vol = _volume(11, 13, 9, rng)
        for dx, dy in DIRS:
            a = b200.aggregate_single_path(vol, img, cfg, intr, dx, dy)
            b = oracle.aggregate_single_path(vol, img, cfg, intr, dx, dy)
            assert_same(a.values, b.values, f"path {dx},{dy}")


STEPS = [(2, 1), (-1, 3), (3, 0), (0, -2), (-2, -2), (4, -3), (20, 0), (0, 0), (1, 0), (-1, 1)]


@pytest.mark.parametrize("group", ["0", "4x3", "4x4", "32x4"])
@pytest.mark.parametrize("variant", [SgmVariant.Plane, SgmVariant.PathGradient])
def test_aggregate_single_path_any_step(b200, oracle, rng, variant, group, monkeypatch):
    """aggregate_single_path walks any integer step (sgm.cpp:210-229): lines
    start at the pixels whose predecessor (x - dx, y - dy) is outside."""
    _blocking(monkeypatch, group)
    w, h = 17, 11
    img = rng.integers(0, 256, (h, w)).astype(np.uint8)
    intr = Intrinsics(30.0, 30.0, 8.0, 5.0, w, h)
    cfg = SgmConfig(variant, 8, 60.0, True, 0.0, 8.0, 10.0, 2)
    vol = _volume(14, w, h, rng)
    for dx, dy in STEPS:
        a = b200.aggregate_single_path(vol, img, cfg, intr, dx, dy)
        b = oracle.aggregate_single_path(vol, img, cfg, intr, dx, dy)
        assert_same(a.values, b.values, f"step {dx},{dy}")


def test_aggregate_single_path_sn_noncanonical(b200, rng):
    """The surface-normal shift exists only for the canonical directions: a
    non-unit step that links two non-empty pixels is a ConfigError
    (sgm.cpp:72-80; the reference throws it from a worker thread)."""
    w, h = 9, 7
    vol = _volume(6, w, h, rng, ragged=False)
    img = rng.integers(0, 256, (h, w)).astype(np.uint8)
    intr = Intrinsics(20.0, 20.0, 4.0, 3.0, w, h)
    pn = np.tile(np.array([0, 0, -1], np.float32), (h, w, 1))
    pd = np.full((h, w), 10.0, np.float32)
    with pytest.raises(ConfigError):
        b200.aggregate_single_path(vol, img, SgmConfig(SgmVariant.SurfaceNormal), intr, 2, 1, pn, pd)


@pytest.mark.parametrize("group", ["0", "4x3", "4x4", "8x2", "32x4"])
@pytest.mark.parametrize("variant", [SgmVariant.Plane, SgmVariant.SurfaceNormal, SgmVariant.PathGradient])
@pytest.mark.parametrize("paths", [8, 4])
def test_aggregate_variants_bitexact(b200, oracle, rng, variant, paths, group, monkeypatch):
    _blocking(monkeypatch, group)
    w, h, planes = 37, 29, 48
    img = rng.integers(0, 256, (h, w)).astype(np.uint8)
    intr = Intrinsics(40.0, 40.0, 18.0, 14.0, w, h)
    vol = _volume(planes, w, h, rng, ragged=True, max_cost=510)
    pn = pd = None
    if variant == SgmVariant.SurfaceNormal:
        nrm = rng.normal(size=(h, w, 3))
        nrm[..., 2] = -np.abs(nrm[..., 2]) - 1.0
        nrm /= np.linalg.norm(nrm, axis=-1, keepdims=True)
        pn = nrm.astype(np.float32)
        pd = rng.uniform(10, 14, (h, w)).astype(np.float32)
        pd[rng.random((h, w)) < 0.1] = 0
    cfg = SgmConfig(variant, paths, 100.0, True, 0.0, 8.0, 10.0, 2)
    a = b200.aggregate(vol, img, cfg, intr, pn, pd)
    b = oracle.aggregate(vol, img, cfg, intr, pn, pd)
    assert_same(a.values, b.values, "aggregate")
    assert_same(b200.wta(a), oracle.wta(b), "wta")


@pytest.mark.parametrize("group", ["4x3", "4x4", "8x4", "32x1", "32x4", "32x8"])
@pytest.mark.parametrize("variant", [SgmVariant.Plane, SgmVariant.PathGradient])
def test_aggregate_dense_wide(b200, oracle, rng, group, variant, monkeypatch):
    """Dense coarsest-level shape: >32 hypotheses per pixel (multi-pass lanes,
    global overflow buffers of the lane-blocked kernel)."""
    _blocking(monkeypatch, group)
    w, h, planes = 40, 24, 130
    img = rng.integers(0, 256, (h, w)).astype(np.uint8)
    intr = Intrinsics(40.0, 40.0, 19.5, 11.5, w, h)
    vol = _volume(planes, w, h, rng, ragged=False, max_cost=510)
    cfg = SgmConfig(variant, 8, 100.0, True, 0.0, 8.0, 10.0, 2)
    a = b200.aggregate(vol, img, cfg, intr)
    b = oracle.aggregate(vol, img, cfg, intr)
    assert_same(a.values, b.values, "aggregate")


def test_aggregate_noncompact_layouts(b200, oracle, rng):
    """The reference layout allows any per-pixel offsets (test_sgm.cpp:262-274
    zeroes a count in place): holes, reversed pixel order and shared trailing
    space are gathered into the compact device layout and scattered back."""
    w, h, planes = 11, 7, 9
    img = rng.integers(0, 256, (h, w)).astype(np.uint8)
    intr = Intrinsics(20.0, 20.0, 5.0, 3.0, w, h)
    cfg = SgmConfig(SgmVariant.Plane, 8, 50.0, True, 0.0, 8.0, 10.0, 2)
    vol = _volume(planes, w, h, rng)
    holes = vol.count.copy()
    holes[rng.random(w * h) < 0.2] = 0
    rev = np.zeros(w * h, np.uint64)
    rev[::-1] = np.cumsum(vol.count[::-1], dtype=np.uint64) - vol.count[::-1].astype(np.uint64)
    pad = np.concatenate([vol.costs, rng.integers(0, 300, 17).astype(np.uint16)])
    cases = [(holes, vol.offset, vol.costs), (vol.count, rev, vol.costs[::-1].copy()),
             (vol.count, vol.offset, pad)]
    for count, offset, costs in cases:
        v = CostVolume(w, h, vol.planes, 2, vol.first, count, offset, costs)
        a = b200.aggregate(v, img, cfg, intr)
        b = oracle.aggregate(v, img, cfg, intr)
        assert_same(a.values, b.values, "aggregate")
        assert_same(b200.wta(b), oracle.wta(b), "wta")
        for dx, dy in ((1, 0), (2, -1)):
            assert_same(b200.aggregate_single_path(v, img, cfg, intr, dx, dy).values,
                        oracle.aggregate_single_path(v, img, cfg, intr, dx, dy).values, "single path")


def test_aggregate_errors(b200, oracle, rng):
    vol = _volume(5, 6, 4, rng)
    img = np.zeros((4, 6), np.uint8)
    intr = Intrinsics(10.0, 10.0, 2.5, 1.5, 6, 4)
    for be in (b200, oracle):
        with pytest.raises(ConfigError):
            be.aggregate(vol, img, SgmConfig(SgmVariant.SurfaceNormal), intr)
        with pytest.raises(ConfigError):
            be.aggregate(vol, img, SgmConfig(paths=6), intr)
        with pytest.raises(ConfigError):
            be.aggregate(vol, img, SgmConfig(phi2_adaptive=False, phi2_fixed=1.0), intr)


def test_normal_offsets_bitexact(b200, oracle, rng):
    w, h = 45, 33
    stack = PlaneStack(harmonic_stack(90, fb=400.0, disp0=20.0))
    intr = Intrinsics(50.0, 52.0, 22.0, 16.5, w, h)
    nrm = rng.normal(size=(h, w, 3))
    nrm[..., 2] = -np.abs(nrm[..., 2]) - 0.5
    nrm /= np.linalg.norm(nrm, axis=-1, keepdims=True)
    nrm = nrm.astype(np.float32)
    nrm[rng.random((h, w)) < 0.05] = 0
    depth = rng.uniform(12, 19, (h, w)).astype(np.float32)
    depth[rng.random((h, w)) < 0.05] = 0
    assert_same(b200.compute_normal_offsets(nrm, depth, stack, intr),
                oracle.compute_normal_offsets(nrm, depth, stack, intr), "offsets")


def test_tail_maps_bitexact(b200, oracle, rng):
    w, h = 61, 47
    intr = Intrinsics(70.0, 71.0, 30.5, 23.0, w, h)
    yy, xx = np.mgrid[0:h, 0:w]
    depth = (8.0 + 0.03 * xx + 0.05 * yy + rng.normal(0, 0.02, (h, w))).astype(np.float32)
    depth[rng.random((h, w)) < 0.08] = 0.0
    assert_same(b200.median_filter_5x5(depth), oracle.median_filter_5x5(depth), "median")
    raw_a = b200.normals_from_depth(depth, intr)
    raw_b = oracle.normals_from_depth(depth, intr)
    assert_same(raw_a, raw_b, "raw normals")
    img = rng.integers(0, 256, (h, w)).astype(np.uint8)
    for r in (1, 2, 3):
        sa = b200.smooth_normals(raw_b, img, r)
        sb = oracle.smooth_normals(raw_b, img, r)
        assert_same(sa, sb, f"smooth r={r}")
    sn = (0.0, -0.2, -np.sqrt(1 - 0.04))
    for rho in (60.0, 45.0):
        assert_same(b200.confidence_map(sb, sn, rho), oracle.confidence_map(sb, sn, rho), "confidence")
    for ow, oh in ((w * 2, h * 2), (w * 2 - 1, h * 2 - 1)):
        assert_same(b200.upscale_nearest(depth, ow, oh), oracle.upscale_nearest(depth, ow, oh), "up d")
        assert_same(b200.upscale_nearest(sb, ow, oh), oracle.upscale_nearest(sb, ow, oh), "up n")


# ---------------------------------------------------------- end to end ----
PKG = __import__("paper_2112_00821_b200")
from conftest import ROOT  # noqa: E402

E2E = [
    # (name, scene kwargs, config kwargs)
    ("c4_fronto_ncc_pi", dict(kind="fronto", w=160, h=120, focal=160.0, depth=10.0, step=0.5, texture=0.35),
     dict(d_min=8.0, d_max=14.0, levels=1, cost="ncc5")),
    ("census_sn_3lvl", dict(kind="slanted", w=192, h=108, focal=192.0, depth=10.0, tilt=30.0, step=0.59,
                            texture=0.2), dict(d_min=4.0, d_max=40.0, levels=3, cost="census5",
                                               variant=SgmVariant.SurfaceNormal, max_planes=128)),
    ("c5_slanted_pg", dict(kind="slanted", w=160, h=60, focal=80.0, depth=5.0, tilt=45.0, step=1.75,
                           texture=0.35), dict(d_min=3.2, d_max=9.0, levels=2, cost="ncc5",
                                               variant=SgmVariant.PathGradient)),
    ("census97_4paths", dict(kind="fronto", w=96, h=80, focal=96.0, depth=10.0, step=0.6, views=3),
     dict(d_min=8.0, d_max=13.0, levels=2, cost="census97", paths=4)),
    ("ncc9_sn_7views", dict(kind="slanted", w=120, h=90, focal=120.0, depth=10.0, tilt=20.0, step=0.4,
                            views=7), dict(d_min=6.0, d_max=20.0, levels=2, cost="ncc9",
                                           variant=SgmVariant.SurfaceNormal)),
    # tilted sweep normal (test_pipeline.cpp:170-182), 3 levels, census + SN
    ("tilted_sweep_census", dict(kind="slanted", w=120, h=90, focal=120.0, depth=8.0, tilt=30.0, step=0.6,
                                 texture=0.4), dict(d_min=5.0, d_max=13.0, levels=2, cost="census5",
                                                    variant=SgmVariant.SurfaceNormal,
                                                    sweep_normal=(0.0, -0.5, -0.8660254037844386))),
    # fixed range policy, fixed phi2, smoothing radius 3, PG
    ("fixed_range_pg", dict(kind="slanted", w=128, h=96, focal=128.0, depth=10.0, tilt=25.0, step=0.5,
                            texture=0.3), dict(d_min=4.0, d_max=30.0, levels=3, cost="census5",
                                               variant=SgmVariant.PathGradient,
                                               range_policy=RangePolicy(RangeKind.Fixed, 0.9),
                                               normal_smoothing_radius=3)),
    # full range policy (every refined pixel sweeps the whole stack: wide pixels)
    ("full_range_ncc", dict(kind="fronto", w=96, h=72, focal=96.0, depth=10.0, step=0.5, texture=0.35),
     dict(d_min=7.0, d_max=15.0, levels=2, cost="ncc5", range_policy=RangePolicy(RangeKind.Full, 0.0))),
    # dense single level with > 128 planes (coarsest-level SGM with K = 8 lanes)
    ("dense_216_planes", dict(kind="slanted", w=96, h=64, focal=400.0, depth=10.0, tilt=20.0, step=1.2,
                              texture=0.3), dict(d_min=4.0, d_max=40.0, levels=1, cost="census5",
                                                 max_planes=256)),
    # fixed phi2, 4 paths, 9 views
    ("fixed_phi2_9views", dict(kind="slanted", w=112, h=84, focal=112.0, depth=10.0, tilt=15.0, step=0.3,
                               views=9), dict(d_min=6.0, d_max=18.0, levels=2, cost="census5",
                                              sgm=SgmConfig(SgmVariant.Plane, 4, 80.0, False, 300.0,
                                                            8.0, 10.0, 1), bundle_size=9)),
]


@pytest.mark.parametrize("group,arena", [("default", None), ("4x4", None), ("8x2", None), ("4x4", "1000")])
@pytest.mark.parametrize("name,scene,cfg", E2E, ids=[e[0] for e in E2E])
def test_estimate_bundle_bitexact(b200, oracle, name, scene, cfg, group, arena, monkeypatch):
    """arena="1000": per-level compact cost-volume arenas (the 4K path);
    group "4x4": K = 4 with u16 costs in 48-byte SGM records, "8x2": the
    general SGM kernel, "default": the library's own blocking."""
    _blocking(monkeypatch, group)
    if arena:
        monkeypatch.setenv("FMVS_ARENA_ENTRIES", arena)
    scene = dict(scene)
    kind = scene.pop("kind")
    bundle, _, _ = render(oracle, kind, **scene)
    c = config(**cfg)
    a = b200.estimate_bundle(bundle, c)
    b = oracle.estimate_bundle(bundle, c)
    assert_same(a.depth, b.depth, "depth")
    assert_same(a.normals, b.normals, "normals")
    assert_same(a.confidence, b.confidence, "confidence")
    assert (b.depth > 0).mean() > 0.5


@pytest.mark.parametrize("cost", ["ncc5", "ncc9"])
@pytest.mark.parametrize("texture", ["scene", "quantized"])
def test_ncc_exact_list_overflow(b200, oracle, rng, cost, texture, monkeypatch):
    """The NCC sweep's batched exact resolution with its lists shrunk to two
    views / two pending entries (FMVS_NCC_SMALL_LISTS, read per call): the
    early resolution, the owner's serial walk on overflow and the dummy items
    of reserved slots all run, results bit-identical."""
    monkeypatch.setenv("FMVS_NCC_SMALL_LISTS", "1")
    bundle, stack = _level_inputs(oracle, w=96, h=64)
    if texture == "quantized":
        for v in bundle:
            v.image = ((v.image // 48) * 48).astype(np.uint8)
    h, w = bundle[2].image.shape
    lo = np.full((h, w), 6.0, np.float32)
    hi = np.full((h, w), 16.0, np.float32)
    spec = {"ncc5": (CostKind.NccTruncated, 5, 5), "ncc9": (CostKind.NccTruncated, 9, 9)}[cost]
    cf = CostFunctionSpec(*spec)
    a = b200.sweep_cost_volume(bundle, 2, stack, lo, hi, cf)
    b = oracle.sweep_cost_volume(bundle, 2, stack, lo, hi, cf)
    assert_same(a.costs, b.costs, "costs")


@pytest.mark.parametrize("name", ["c4_fronto_ncc_pi", "ncc9_sn_7views"])
def test_estimate_bundle_ncc_small_lists(b200, oracle, name, monkeypatch):
    """Whole bundles (dense and refined levels) through the shrunk NCC lists."""
    monkeypatch.setenv("FMVS_NCC_SMALL_LISTS", "1")
    _, scene, cfg = next(e for e in E2E if e[0] == name)
    scene = dict(scene)
    kind = scene.pop("kind")
    bundle, _, _ = render(oracle, kind, **scene)
    c = config(**cfg)
    a = b200.estimate_bundle(bundle, c)
    b = oracle.estimate_bundle(bundle, c)
    assert_same(a.depth, b.depth, "depth")
    assert_same(a.normals, b.normals, "normals")
    assert_same(a.confidence, b.confidence, "confidence")


@pytest.mark.parametrize("name", ["dense_216_planes", "c4_fronto_ncc_pi", "census_sn_3lvl", "c5_slanted_pg"])
def test_estimate_bundle_packed_aggregate(oracle, name, monkeypatch):
    """The packed u16 SGM aggregate (two entries per 32-bit RED word), which
    the library uses on uniform levels too large for L2 (C3, C4), forced on
    small uniform levels: results bit-identical."""
    monkeypatch.setenv("FMVS_SGM_AGG16_MIN", "0")
    # a context of its own, created with the hook set (not the shared one)
    b200 = PKG.Backend(os.path.join(ROOT, "paper_2112_00821_b200", "_lib", "libfmvs.so"), "fmvs_", 0)
    try:
        _, scene, cfg = next(e for e in E2E if e[0] == name)
        scene = dict(scene)
        kind = scene.pop("kind")
        bundle, _, _ = render(oracle, kind, **scene)
        c = config(**cfg)
        a = b200.estimate_bundle(bundle, c)
        b = oracle.estimate_bundle(bundle, c)
        assert_same(a.depth, b.depth, "depth")
        assert_same(a.normals, b.normals, "normals")
        assert_same(a.confidence, b.confidence, "confidence")
        cap = b200.estimate_bundle_captured(bundle, c, level=c.pyramid_levels - 1)
        ref = oracle.estimate_bundle_captured(bundle, c, level=c.pyramid_levels - 1)
        assert_same(cap["aggregate"], ref["aggregate"], "coarsest-level aggregate")
    finally:
        b200.close()


def test_estimate_bundle_deterministic(b200, oracle):
    bundle, _, _ = render(oracle, "slanted", 128, 96, tilt=30.0)
    c = config(4.0, 40.0, levels=3, cost="census5", variant=SgmVariant.SurfaceNormal)
    a = b200.estimate_bundle(bundle, c)
    b = b200.estimate_bundle(bundle, c)
    assert_same(a.depth, b.depth, "depth")
    assert_same(a.normals, b.normals, "normals")


def test_estimate_bundle_errors_match(b200, oracle):
    bundle, _, _ = render(oracle, "fronto", 48, 32)
    cases = [
        (bundle[:4], config(8.0, 14.0), InvalidInputError),               # even bundle
        (bundle, config(8.0, 14.0, variant=SgmVariant.SurfaceNormal), ConfigError),  # SN needs 2 levels
        (bundle, config(8.0, 14.0, bundle_size=4), ConfigError),
        (bundle, config(8.0, 14.0, max_planes=1), ConfigError),
        (bundle, config(8.0, 14.0, normal_smoothing_radius=0), ConfigError),
    ]
    for bnd, c, exc in cases:
        for be in (b200, oracle):
            with pytest.raises(exc):
                be.estimate_bundle(bnd, c)
    # zero baseline -> GeometryError (test_pipeline.cpp:198-205)
    flat = [type(v)(v.image, v.intrinsics, type(v.pose)(v.pose.rotation, np.zeros(3))) for v in bundle]
    for be in (b200, oracle):
        with pytest.raises(GeometryError):
            be.estimate_bundle(flat, config(8.0, 14.0))


@pytest.mark.parametrize("case", ["cropped_views", "tiny_3lvl", "odd_sizes"])
def test_estimate_bundle_shapes(b200, oracle, case):
    """Matching views of different sizes than the reference (cropped
    right/bottom, intrinsics kept), tiny images whose coarsest level is a few
    pixels, and odd sizes (ceil-halving pyramid)."""
    import dataclasses
    if case == "cropped_views":
        bundle, _, _ = render(oracle, "slanted", 120, 90, tilt=25.0, step=0.5, texture=0.3)
        for k in (0, 1, 3, 4):
            v = bundle[k]
            cw, ch = 120 - 7 * (k + 1), 90 - 3 * k
            v.image = np.ascontiguousarray(v.image[:ch, :cw])
            v.intrinsics = dataclasses.replace(v.intrinsics, width=cw, height=ch)
        c = config(4.0, 40.0, levels=2, cost="census5", variant=SgmVariant.SurfaceNormal, max_planes=64)
    elif case == "tiny_3lvl":
        bundle, _, _ = render(oracle, "fronto", 13, 9, focal=13.0, step=0.3, texture=0.5)
        c = config(6.0, 16.0, levels=3, cost="ncc5", max_planes=32)
    else:
        bundle, _, _ = render(oracle, "slanted", 101, 77, tilt=20.0, step=0.45, texture=0.3)
        c = config(4.0, 30.0, levels=3, cost="census97", variant=SgmVariant.PathGradient, max_planes=48)
    a = b200.estimate_bundle(bundle, c)
    b = oracle.estimate_bundle(bundle, c)
    assert_same(a.depth, b.depth, "depth")
    assert_same(a.normals, b.normals, "normals")
    assert_same(a.confidence, b.confidence, "confidence")


def test_contexts_on_concurrent_host_threads(oracle):
    """One context per host thread, bundles of different configurations
    (level sizes, plane counts, SGM variants, census / NCC) launched
    concurrently: every result bit-identical to the oracle's. Guards the
    per-kernel launch attributes that concurrent contexts share."""
    import threading
    cases = [E2E[i] for i in (0, 1, 2, 6, 8)]
    inputs = []
    for name, scene, cfg in cases:
        scene = dict(scene)
        kind = scene.pop("kind")
        bundle, _, _ = render(oracle, kind, **scene)
        c = config(**cfg)
        inputs.append((name, bundle, c, oracle.estimate_bundle(bundle, c)))
    path = os.path.join(ROOT, "paper_2112_00821_b200", "_lib", "libfmvs.so")
    errors = []

    def worker(k):
        b = PKG.Backend(path, "fmvs_", 0)
        try:
            for rep in range(3):
                for j in range(len(inputs)):
                    name, bundle, c, want = inputs[(j + k) % len(inputs)]
                    got = b.estimate_bundle(bundle, c)
                    if not (np.array_equal(got.depth, want.depth) and np.array_equal(got.normals, want.normals)
                            and np.array_equal(got.confidence, want.confidence)):
                        errors.append(f"thread {k} rep {rep}: {name} differs")
        except Exception as e:  # reported below
            errors.append(f"thread {k}: {type(e).__name__}: {e}")
        finally:
            b.close()

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
