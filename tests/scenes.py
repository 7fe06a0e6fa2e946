"""Seeded synthetic bundles shared by the tests (rendered by the oracle's
render_scene, render.cpp:52-141, so both implementations see identical
bytes), and small config builders mirroring the acceptance criteria."""
from __future__ import annotations

import numpy as np

from paper_2112_00821_b200 import (CalibratedView, CostFunctionSpec, CostKind, Intrinsics,
                                   PipelineConfig, Pose, SgmConfig, SgmVariant)


def render(backend, kind="fronto", w=160, h=120, focal=None, depth=10.0, views=5, step=0.5,
           seed=1, tilt=0.0, texture=0.35):
    focal = float(w) if focal is None else focal
    return backend.render_plane_scene(kind, w, h, focal, depth, views, step, seed=seed,
                                      tilt_deg=tilt, texture_scale=texture)


def config(d_min, d_max, levels=1, cost="ncc5", variant=SgmVariant.Plane, paths=8,
           max_planes=256, **kw) -> PipelineConfig:
    kinds = {"ncc5": (CostKind.NccTruncated, 5, 5), "ncc9": (CostKind.NccTruncated, 9, 9),
             "census5": (CostKind.CensusHamming, 5, 5), "census97": (CostKind.CensusHamming, 9, 7)}
    k, ww, wh = kinds[cost]
    c = PipelineConfig(d_min, d_max, pyramid_levels=levels, max_planes=max_planes,
                       sgm=SgmConfig(variant=variant, paths=paths),
                       cost=CostFunctionSpec(k, ww, wh))
    for key, val in kw.items():
        setattr(c, key, val)
    return c


def rotation(rng, max_angle):
    axis = rng.uniform(-1, 1, 3)
    axis /= np.linalg.norm(axis)
    a = rng.uniform(0, max_angle)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + np.sin(a) * K + (1 - np.cos(a)) * K @ K


def random_camera_pair(rng, w=64, h=48):
    k = Intrinsics(float(rng.uniform(50, 120)), float(rng.uniform(50, 120)),
                   (w - 1) / 2.0 + rng.uniform(-3, 3), (h - 1) / 2.0 + rng.uniform(-3, 3), w, h)
    ref = Pose(rotation(rng, 0.05), rng.uniform(-0.1, 0.1, 3))
    other = Pose(rotation(rng, 0.1), ref.center + np.array([rng.uniform(0.3, 1.0), rng.uniform(-0.2, 0.2),
                                                            rng.uniform(-0.1, 0.1)]))
    return k, ref, other


def random_volume(rng, w, h, planes, ragged=True, max_cost=300):
    """random_volume of test_sgm.cpp:25-55 (numpy RNG)."""
    first = np.zeros(w * h, np.int32)
    count = np.full(w * h, planes, np.int32)
    if ragged:
        first = rng.integers(0, planes, w * h).astype(np.int32)
        count = np.array([rng.integers(0, planes - f + 1) for f in first], np.int32)
    offset = np.zeros(w * h, np.uint64)
    offset[1:] = np.cumsum(count[:-1], dtype=np.uint64)
    costs = rng.integers(0, max_cost + 1, int(count.sum())).astype(np.uint16)
    return first, count, offset, costs


def harmonic_stack(count, fb=300.0, disp0=20.0):
    return np.array([fb / (disp0 + i) for i in range(count)], np.float64)
