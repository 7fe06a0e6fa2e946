"""Python mirror of the reference's public API (proj/include/fassmvs/*.hpp)
over the C ABI (include/fmvs.h).

Same names, argument meaning and error behaviour as the reference:
``estimate_bundle(bundle, config) -> BundleResult`` (pipeline.hpp:79-80),
the stage functions (sweep_cost_volume, aggregate, aggregate_single_path, wta,
compute_normal_offsets, build_pyramids, refine_range, median_filter_5x5,
normals_from_depth, smooth_normals, confidence_map, upscale_nearest, the
host geometry helpers) and the three exception types of errors.hpp:10-24.

A :class:`Backend` binds one shared library. ``Backend.b200()`` is the
product (the in-tree ``_lib/libfmvs.so``, hand-written sm_100a kernels); the
tests also bind the reference oracle through the same class.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _abi


# ------------------------------------------------------------ errors ------
class FassmvsError(RuntimeError):
    pass


class InvalidInputError(FassmvsError):
    """fassmvs::InvalidInputError (errors.hpp:10-13), CLI exit code 1."""


class ConfigError(FassmvsError):
    """fassmvs::ConfigError (errors.hpp:15-19), CLI exit code 2."""


class GeometryError(FassmvsError):
    """fassmvs::GeometryError (errors.hpp:21-24), CLI exit code 1."""


class CudaError(FassmvsError):
    """Device failure (no reference analogue)."""


class CapacityError(FassmvsError):
    """Output buffer too small (C ABI only)."""


_ERRORS = {
    _abi.FMVS_ERR_INVALID_INPUT: InvalidInputError,
    _abi.FMVS_ERR_CONFIG: ConfigError,
    _abi.FMVS_ERR_GEOMETRY: GeometryError,
    _abi.FMVS_ERR_CUDA: CudaError,
    _abi.FMVS_ERR_CAPACITY: CapacityError,
}


# ------------------------------------------------------------- types ------
class CostKind(enum.IntEnum):
    CensusHamming = 0
    NccTruncated = 1


class SgmVariant(enum.IntEnum):
    Plane = 0
    SurfaceNormal = 1
    PathGradient = 2


class RangeKind(enum.IntEnum):
    Full = 0
    Fixed = 1
    SpacingMultiple = 2


@dataclass
class Intrinsics:  # geometry.hpp:19-39
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def to_c(self) -> _abi.Intrinsics_c:
        return _abi.Intrinsics_c(self.fx, self.fy, self.cx, self.cy, self.width, self.height)

    @staticmethod
    def from_c(c: _abi.Intrinsics_c) -> "Intrinsics":
        return Intrinsics(c.fx, c.fy, c.cx, c.cy, c.width, c.height)

    def halved(self) -> "Intrinsics":  # geometry.cpp:30-39
        return Intrinsics(self.fx / 2.0, self.fy / 2.0, self.cx / 2.0, self.cy / 2.0,
                          (self.width + 1) // 2, (self.height + 1) // 2)


@dataclass
class Pose:  # geometry.hpp:44-55
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    center: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def to_c(self) -> _abi.Pose_c:
        p = _abi.Pose_c()
        r = np.asarray(self.rotation, dtype=np.float64).reshape(9)
        c = np.asarray(self.center, dtype=np.float64).reshape(3)
        for i in range(9):
            p.rotation[i] = float(r[i])
        for i in range(3):
            p.center[i] = float(c[i])
        return p

    @staticmethod
    def from_c(c: _abi.Pose_c) -> "Pose":
        return Pose(np.array(list(c.rotation), dtype=np.float64).reshape(3, 3),
                    np.array(list(c.center), dtype=np.float64))


@dataclass
class CalibratedView:  # geometry.hpp:57-63
    image: np.ndarray  # uint8 (height, width)
    intrinsics: Intrinsics
    pose: Pose


@dataclass
class PlaneStack:  # geometry.hpp:75-94
    distances: np.ndarray
    normal: tuple = (0.0, 0.0, -1.0)

    def count(self) -> int:
        return int(len(self.distances))


@dataclass
class SgmConfig:  # sgm.hpp:19-32
    variant: SgmVariant = SgmVariant.Plane
    paths: int = 8
    phi1: float = 100.0
    phi2_adaptive: bool = True
    phi2_fixed: float = 0.0
    alpha: float = 8.0
    beta: float = 10.0
    penalty_scale: int = 1

    def to_c(self) -> _abi.SgmConfig_c:
        return _abi.SgmConfig_c(int(self.variant), self.paths, self.phi1, int(bool(self.phi2_adaptive)),
                                self.phi2_fixed, self.alpha, self.beta, self.penalty_scale)


@dataclass
class CostFunctionSpec:  # matching.hpp:14-23
    kind: CostKind = CostKind.NccTruncated
    window_w: int = 5
    window_h: int = 5

    def to_c(self) -> _abi.CostSpec_c:
        return _abi.CostSpec_c(int(self.kind), self.window_w, self.window_h)

    def census_bits(self) -> int:
        return self.window_w * self.window_h - 1


@dataclass
class RangePolicy:  # pipeline.hpp:12-20
    kind: RangeKind = RangeKind.SpacingMultiple
    value: float = 3.0


@dataclass
class PipelineConfig:  # pipeline.hpp:22-35
    d_min: float
    d_max: float
    bundle_size: int = 5
    pyramid_levels: int = 3
    sweep_normal: tuple = (0.0, 0.0, -1.0)
    range_policy: RangePolicy = field(default_factory=RangePolicy)
    max_planes: int = 256
    sgm: SgmConfig = field(default_factory=SgmConfig)
    cost: CostFunctionSpec = field(default_factory=CostFunctionSpec)
    normal_smoothing_radius: int = 2

    def to_c(self) -> _abi.Config_c:
        c = _abi.Config_c()
        c.bundle_size = self.bundle_size
        c.pyramid_levels = self.pyramid_levels
        c.d_min = self.d_min
        c.d_max = self.d_max
        for i in range(3):
            c.sweep_normal[i] = float(self.sweep_normal[i])
        c.range_kind = int(self.range_policy.kind)
        c.range_value = float(self.range_policy.value)
        c.max_planes = self.max_planes
        c.sgm = self.sgm.to_c()
        c.cost = self.cost.to_c()
        c.normal_smoothing_radius = self.normal_smoothing_radius
        return c


@dataclass
class BundleResult:  # pipeline.hpp:37-41
    depth: np.ndarray       # float32 (h, w)
    normals: np.ndarray     # float32 (h, w, 3)
    confidence: np.ndarray  # float32 (h, w)


@dataclass
class CostVolume:  # matching.hpp:36-53
    width: int
    height: int
    planes: PlaneStack
    per_side: int
    first: np.ndarray   # int32 (h*w)
    count: np.ndarray   # int32 (h*w)
    offset: np.ndarray  # uint64 (h*w)
    costs: np.ndarray   # uint16 (total)

    def pixel_costs(self, x: int, y: int) -> np.ndarray:
        p = y * self.width + x
        return self.costs[int(self.offset[p]):int(self.offset[p]) + int(self.count[p])]


@dataclass
class AggregatedVolume:  # sgm.hpp:39-49
    width: int
    height: int
    planes: PlaneStack
    first: np.ndarray
    count: np.ndarray
    offset: np.ndarray
    values: np.ndarray  # uint32 (total)


class DepthLookup(enum.IntEnum):  # postfilter.hpp:30
    Nearest = 0
    Bilinear = 1


@dataclass
class GeomFilterConfig:  # postfilter.hpp:32-36
    eta_r: float = 10.0
    eta_h: int = 3
    lookup: DepthLookup = DepthLookup.Nearest

    def to_c(self) -> _abi.GeomFilterConfig_c:
        return _abi.GeomFilterConfig_c(float(self.eta_r), int(self.eta_h), int(self.lookup))


@dataclass
class ConsistencyView:  # postfilter.hpp:24-28
    depth: np.ndarray       # float32 (h, w)
    intrinsics: "Intrinsics"
    pose: "Pose"


class Filter(enum.IntEnum):  # the CLI's --filter (tools/fassmvs.cpp:97-99)
    none = 0
    dog = 1
    geom = 2
    both = 3


@dataclass
class FrameResult:  # tools/fassmvs.cpp:140-143
    frame: int
    maps: BundleResult


# ----------------------------------------------------------- helpers ------
def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _pd(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _stack_c(planes: PlaneStack):
    d = np.ascontiguousarray(planes.distances, dtype=np.float64)
    s = _abi.PlaneStack_c()
    for i in range(3):
        s.normal[i] = float(planes.normal[i])
    s.distances = d.ctypes.data_as(C.c_void_p)
    s.count = len(d)
    return s, d


def _views_c(bundle: Sequence[CalibratedView]):
    arr = (_abi.View_c * max(1, len(bundle)))()
    keep = []
    for i, v in enumerate(bundle):
        img = np.ascontiguousarray(v.image, dtype=np.uint8)
        keep.append(img)
        arr[i].image = img.ctypes.data_as(C.c_void_p)
        arr[i].intrinsics = v.intrinsics.to_c()
        arr[i].pose = v.pose.to_c()
    return arr, keep


def _f32(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float32)
    if shape is not None:
        out = out.reshape(shape)
    return out


# ----------------------------------------------------------- backend ------
class Backend:
    """One bound library (the B200 product or, in tests, the oracle)."""

    def __init__(self, lib_path: str, prefix: str, device: int = 0, extras: dict | None = None,
                 needs_context: bool = True):
        if not os.path.exists(lib_path):
            raise FileNotFoundError(lib_path)
        self.path = lib_path
        self.lib = C.CDLL(lib_path)
        self.prefix = prefix
        self.fn = _abi.bind(self.lib, prefix, extras)
        self.ctx = C.c_void_p()
        if needs_context:
            self._check(self.fn["ctx_create"](device, C.byref(self.ctx)))

    _b200_singleton: "Backend | None" = None

    @classmethod
    def b200(cls, device: int = 0) -> "Backend":
        """The product library; fails loudly when the CUDA build is missing."""
        if device == 0 and cls._b200_singleton is not None:
            return cls._b200_singleton
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libfmvs.so")
        if not os.path.exists(path):
            raise RuntimeError(
                f"B200 library not built ({path}); run __graft_entry__.build() or "
                "make -C paper_2112_00821_b200")
        b = cls(path, "fmvs_", device)
        if device == 0:
            cls._b200_singleton = b
        return b

    def close(self):
        if self.ctx and "ctx_destroy" in self.fn:
            self.fn["ctx_destroy"](self.ctx)
            self.ctx = C.c_void_p()

    # -- plumbing
    def _check(self, rc: int):
        if rc != _abi.FMVS_OK:
            msg = self.fn["last_error"]().decode(errors="replace")
            raise _ERRORS.get(rc, FassmvsError)(msg)

    def last_error(self) -> str:
        return self.fn["last_error"]().decode(errors="replace")

    # ------------------------------------------------------------ hot path
    def estimate_bundle(self, bundle: Sequence[CalibratedView], config: PipelineConfig) -> BundleResult:
        """estimate_bundle (pipeline.hpp:79-80)."""
        views, keep = _views_c(bundle)
        cfg = config.to_c()
        n = len(bundle)
        ref = bundle[n // 2] if n else None
        w = ref.intrinsics.width if ref is not None else 1
        h = ref.intrinsics.height if ref is not None else 1
        w, h = max(w, 1), max(h, 1)
        depth = np.zeros((h, w), np.float32)
        normals = np.zeros((h, w, 3), np.float32)
        conf = np.zeros((h, w), np.float32)
        self._check(self.fn["estimate_bundle"](self.ctx, views, n, C.byref(cfg), _ptr(depth),
                                               _ptr(normals), _ptr(conf)))
        del keep
        return BundleResult(depth, normals, conf)

    def estimate_bundle_captured(self, bundle: Sequence[CalibratedView], config: PipelineConfig,
                                 level: int = 0) -> dict:
        """estimate_bundle keeping one level's intermediates (parity debugging):
        the ragged layout first/count/offset of the reference's CostVolume
        (matching.hpp:36-53), u16 costs, u32 aggregate, WTA winners and the
        depth before the median filter (pipeline.cpp:263-288)."""
        self._check(self.fn["ctx_set_capture"](self.ctx, level))
        res = self.estimate_bundle(bundle, config)
        w, h, n = C.c_int32(), C.c_int32(), C.c_uint64()
        self._check(self.fn["ctx_capture_sizes"](self.ctx, C.byref(w), C.byref(h), C.byref(n)))
        px = w.value * h.value
        out = dict(first=np.zeros(px, np.int32), count=np.zeros(px, np.int32),
                   offset=np.zeros(px, np.uint64), costs=np.zeros(n.value, np.uint16),
                   aggregate=np.zeros(n.value, np.uint32), winners=np.zeros(px, np.int32),
                   depth_raw=np.zeros((h.value, w.value), np.float32))
        self._check(self.fn["ctx_capture_copy"](
            self.ctx, *(_ptr(out[k]) for k in ("first", "count", "offset", "costs", "aggregate",
                                               "winners", "depth_raw"))))
        self.fn["ctx_set_capture"](self.ctx, -1)
        out["result"] = res
        return out

    def level_stats(self):
        out = (_abi.LevelStats_c * 16)()
        n = self.fn["ctx_level_stats"](self.ctx, out, 16)
        return [dict(width=out[i].width, height=out[i].height, planes=out[i].planes,
                     entries=int(out[i].entries)) for i in range(n)]

    def last_launch_count(self) -> int:
        return int(self.fn["ctx_last_launch_count"](self.ctx))

    # ------------------------------------------------------ host geometry
    def plane_homography(self, normal, distance, ref_intr: Intrinsics, ref_pose: Pose,
                         other_intr: Intrinsics, other_pose: Pose) -> np.ndarray:
        n = np.asarray(normal, np.float64)
        out = np.zeros(9, np.float64)
        self._check(self.fn["plane_homography"](_pd(n), float(distance), C.byref(ref_intr.to_c()),
                                                C.byref(ref_pose.to_c()), C.byref(other_intr.to_c()),
                                                C.byref(other_pose.to_c()), _pd(out)))
        return out.reshape(3, 3)

    def bounding_distances(self, d_min, d_max, normal, ref_intr: Intrinsics):
        n = np.asarray(normal, np.float64)
        lo, hi = C.c_double(), C.c_double()
        self._check(self.fn["bounding_distances"](d_min, d_max, _pd(n), C.byref(ref_intr.to_c()),
                                                  C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def plane_distances(self, ref_intr, ref_pose, other_intr, other_pose, delta_min, delta_max,
                        normal, max_planes) -> np.ndarray:
        n = np.asarray(normal, np.float64)
        cap = 4096
        while True:
            out = np.zeros(cap, np.float64)
            cnt = C.c_int32()
            rc = self.fn["plane_distances"](C.byref(ref_intr.to_c()), C.byref(ref_pose.to_c()),
                                            C.byref(other_intr.to_c()), C.byref(other_pose.to_c()),
                                            delta_min, delta_max, _pd(n), max_planes, _pd(out), cap,
                                            C.byref(cnt))
            if rc == _abi.FMVS_ERR_CAPACITY:
                cap = cnt.value
                continue
            self._check(rc)
            return out[:cnt.value].copy()

    def depth_from_plane(self, x, y, normal, distance, intr: Intrinsics) -> float:
        n = np.asarray(normal, np.float64)
        return self.fn["depth_from_plane"](x, y, _pd(n), distance, C.byref(intr.to_c()))

    def adaptive_phi2(self, phi1, alpha, beta, di) -> float:
        return self.fn["adaptive_phi2"](phi1, alpha, beta, di)

    def parabola_refine(self, d_prev, d_win, d_next, c_prev, c_win, c_next) -> float:
        out = C.c_double()
        self._check(self.fn["parabola_refine"](d_prev, d_win, d_next, c_prev, c_win, c_next,
                                               C.byref(out)))
        return out.value

    # ------------------------------------------------------------ stages
    def build_pyramids(self, bundle: Sequence[CalibratedView], levels: int):
        """build_pyramids (pipeline.hpp:50): list of levels of CalibratedView."""
        views, keep = _views_c(bundle)
        n = len(bundle)
        intr = (_abi.Intrinsics_c * max(1, n * max(levels, 1)))()
        cap = sum(int(v.image.size) for v in bundle) * 2 + 16
        out = np.zeros(cap, np.uint8)
        self._check(self.fn["build_pyramids"](self.ctx, views, n, levels, _ptr(out), cap, intr))
        res, pos = [], 0
        for l in range(levels):
            lvl = []
            for k in range(n):
                ki = Intrinsics.from_c(intr[l * n + k])
                px = ki.width * ki.height
                lvl.append(CalibratedView(out[pos:pos + px].reshape(ki.height, ki.width).copy(), ki,
                                          bundle[k].pose))
                pos += px
            res.append(lvl)
        del keep
        return res

    def refine_range(self, prior: np.ndarray, policy: RangePolicy, d_min: float, d_max: float,
                     coarser: Optional[PlaneStack] = None, intrinsics: Optional[Intrinsics] = None):
        prior = _f32(prior)
        h, w = prior.shape
        lo = np.zeros((h, w), np.float32)
        hi = np.zeros((h, w), np.float32)
        st, keep = (_stack_c(coarser) if coarser is not None else (None, None))
        self._check(self.fn["refine_range"](self.ctx, _ptr(prior), w, h, int(policy.kind), policy.value,
                                            d_min, d_max, C.byref(st) if st is not None else None,
                                            C.byref(intrinsics.to_c()) if intrinsics else None,
                                            _ptr(lo), _ptr(hi)))
        return lo, hi

    def sweep_cost_volume(self, bundle: Sequence[CalibratedView], ref_index: int, planes: PlaneStack,
                          lo: np.ndarray, hi: np.ndarray, costfn: CostFunctionSpec) -> CostVolume:
        views, keep = _views_c(bundle)
        n = len(bundle)
        ref = bundle[min(max(ref_index, 0), max(n - 1, 0))]
        w, h = ref.intrinsics.width, ref.intrinsics.height
        px = w * h
        lo = _f32(lo).reshape(-1)
        hi = _f32(hi).reshape(-1)
        first = np.zeros(px, np.int32)
        count = np.zeros(px, np.int32)
        offset = np.zeros(px, np.uint64)
        st, dkeep = _stack_c(planes)
        cap = max(1, px * planes.count())
        costs = np.zeros(cap, np.uint16)
        total = C.c_uint64()
        per_side = C.c_int32()
        cs = costfn.to_c()
        self._check(self.fn["sweep_cost_volume"](self.ctx, views, n, ref_index, C.byref(st), _ptr(lo),
                                                 _ptr(hi), C.byref(cs), _ptr(first), _ptr(count),
                                                 _ptr(offset), _ptr(costs), cap, C.byref(total),
                                                 C.byref(per_side)))
        return CostVolume(w, h, planes, per_side.value, first, count, offset,
                          costs[:total.value].copy())

    def compute_normal_offsets(self, prior_normals: np.ndarray, prior_depth: np.ndarray,
                               planes: PlaneStack, intrinsics: Intrinsics) -> np.ndarray:
        pn = _f32(prior_normals)
        pd = _f32(prior_depth)
        h, w = pd.shape
        out = np.zeros((h, w, 4), np.int16)
        st, keep = _stack_c(planes)
        self._check(self.fn["compute_normal_offsets"](self.ctx, _ptr(pn), _ptr(pd), w, h, C.byref(st),
                                                      C.byref(intrinsics.to_c()), _ptr(out)))
        return out

    def _aggregate(self, vol: CostVolume, image: np.ndarray, config: SgmConfig,
                   intrinsics: Intrinsics, dx: int, dy: int, prior_normals=None, prior_depth=None,
                   entry="aggregate"):
        st, keep = _stack_c(vol.planes)
        img = np.ascontiguousarray(image, np.uint8)
        first = np.ascontiguousarray(vol.first, np.int32)
        count = np.ascontiguousarray(vol.count, np.int32)
        offset = np.ascontiguousarray(vol.offset, np.uint64)
        costs = np.ascontiguousarray(vol.costs, np.uint16)
        out = np.zeros(max(1, len(costs)), np.uint32)
        pn = _f32(prior_normals) if prior_normals is not None else None
        pd = _f32(prior_depth) if prior_depth is not None else None
        cfg = config.to_c()
        self._check(self.fn[entry](self.ctx, vol.width, vol.height, C.byref(st), _ptr(first),
                                   _ptr(count), _ptr(offset), _ptr(costs), len(costs), _ptr(img),
                                   C.byref(cfg), C.byref(intrinsics.to_c()), _ptr(pn), _ptr(pd),
                                   dx, dy, _ptr(out)))
        return AggregatedVolume(vol.width, vol.height, vol.planes, first, count, offset,
                                out[:len(costs)].copy())

    def aggregate(self, vol: CostVolume, image, config: SgmConfig, intrinsics: Intrinsics,
                  prior_normals=None, prior_depth=None) -> AggregatedVolume:
        """aggregate (sgm.hpp:86-89)."""
        return self._aggregate(vol, image, config, intrinsics, 0, 0, prior_normals, prior_depth)

    def aggregate_single_path(self, vol: CostVolume, image, config: SgmConfig, intrinsics: Intrinsics,
                              dir_x: int, dir_y: int, prior_normals=None,
                              prior_depth=None) -> AggregatedVolume:
        """aggregate_single_path (sgm.hpp:91-96): any integer step (dir_x, dir_y)."""
        return self._aggregate(vol, image, config, intrinsics, dir_x, dir_y, prior_normals, prior_depth,
                               entry="aggregate_single_path")

    def wta(self, agg: AggregatedVolume) -> np.ndarray:
        px = agg.width * agg.height
        out = np.zeros(px, np.int32)
        first = np.ascontiguousarray(agg.first, np.int32)
        count = np.ascontiguousarray(agg.count, np.int32)
        offset = np.ascontiguousarray(agg.offset, np.uint64)
        vals = np.ascontiguousarray(agg.values, np.uint32)
        self._check(self.fn["wta"](self.ctx, agg.width, agg.height, _ptr(first), _ptr(count),
                                   _ptr(offset), _ptr(vals), len(vals), _ptr(out)))
        return out.reshape(agg.height, agg.width)

    def median_filter_5x5(self, depth: np.ndarray) -> np.ndarray:
        d = _f32(depth)
        h, w = d.shape
        out = np.zeros_like(d)
        self._check(self.fn["median_filter_5x5"](self.ctx, _ptr(d), w, h, _ptr(out)))
        return out

    def normals_from_depth(self, depth: np.ndarray, intrinsics: Intrinsics) -> np.ndarray:
        d = _f32(depth)
        h, w = d.shape
        out = np.zeros((h, w, 3), np.float32)
        self._check(self.fn["normals_from_depth"](self.ctx, _ptr(d), w, h, C.byref(intrinsics.to_c()),
                                                  _ptr(out)))
        return out

    def smooth_normals(self, raw: np.ndarray, image: np.ndarray, radius: int) -> np.ndarray:
        r = _f32(raw)
        img = np.ascontiguousarray(image, np.uint8)
        h, w = img.shape
        out = np.zeros((h, w, 3), np.float32)
        self._check(self.fn["smooth_normals"](self.ctx, _ptr(r), _ptr(img), w, h, radius, _ptr(out)))
        return out

    def confidence_map(self, normals: np.ndarray, sweep_normal=(0.0, 0.0, -1.0),
                       rho_degrees: float = 60.0) -> np.ndarray:
        nm = _f32(normals)
        h, w = nm.shape[:2]
        out = np.zeros((h, w), np.float32)
        sn = np.asarray(sweep_normal, np.float64)
        self._check(self.fn["confidence_map"](self.ctx, _ptr(nm), w, h, _pd(sn), rho_degrees, _ptr(out)))
        return out

    def upscale_nearest(self, m: np.ndarray, width: int, height: int) -> np.ndarray:
        a = _f32(m)
        ih, iw = a.shape[:2]
        ch = 1 if a.ndim == 2 else a.shape[2]
        out = np.zeros((height, width) + (() if ch == 1 else (ch,)), np.float32)
        self._check(self.fn["upscale_nearest"](self.ctx, _ptr(a), iw, ih, ch, width, height, _ptr(out)))
        return out

    # -------------------------------------------- post-filters (§8f)
    def dog_mask(self, image: np.ndarray) -> np.ndarray:
        """dog_mask (postfilter.hpp:18): uint8 (h, w), 1 = textured."""
        img = np.ascontiguousarray(image, np.uint8)
        h, w = img.shape
        out = np.zeros((h, w), np.uint8)
        self._check(self.fn["dog_mask"](self.ctx, _ptr(img), w, h, _ptr(out)))
        return out

    def apply_mask(self, depth: np.ndarray, normals: np.ndarray, confidence: np.ndarray,
                   mask: np.ndarray) -> BundleResult:
        """apply_mask (postfilter.hpp:21-22); returns the masked maps."""
        d, n, c = _f32(depth).copy(), _f32(normals).copy(), _f32(confidence).copy()
        m = np.ascontiguousarray(mask, np.uint8)
        h, w = d.shape
        if n.shape[:2] != (h, w) or c.shape != (h, w) or m.shape != (h, w):
            raise InvalidInputError("apply mask: map sizes differ")
        self._check(self.fn["apply_mask"](self.ctx, _ptr(d), _ptr(n), _ptr(c), w, h, _ptr(m)))
        return BundleResult(d, n, c)

    def geometric_consistency_mask(self, window: Sequence[ConsistencyView], ref_index: int,
                                   config: GeomFilterConfig | None = None) -> np.ndarray:
        """geometric_consistency_mask (postfilter.hpp:44-45): uint8 keep mask."""
        cfg = (config or GeomFilterConfig()).to_c()
        arr = (_abi.ConsistencyView_c * max(1, len(window)))()
        keep = []
        for i, v in enumerate(window):
            d = _f32(v.depth)
            keep.append(d)
            arr[i].depth = _ptr(d)
            arr[i].height, arr[i].width = d.shape
            arr[i].intrinsics = v.intrinsics.to_c()
            arr[i].pose = v.pose.to_c()
        shape = window[ref_index].depth.shape if 0 <= ref_index < len(window) else (1, 1)
        out = np.zeros(shape, np.uint8)
        self._check(self.fn["geometric_consistency_mask"](self.ctx, arr, len(window), ref_index,
                                                          C.byref(cfg), _ptr(out)))
        del keep
        return out

    def estimate_sequence(self, frames: Sequence[CalibratedView], config: PipelineConfig,
                          stride: int = 1, filter: Filter = Filter.none) -> list:
        """The `fassmvs estimate` loop (tools/fassmvs.cpp:92-176) without file
        I/O: list of FrameResult(frame, maps) for ref = half, half+stride, ..."""
        views, keep = _views_c(frames)
        cfg = config.to_c()
        n = len(frames)
        h, w = (frames[0].image.shape if n else (1, 1))
        half = max(config.bundle_size, 1) // 2
        cap = max(1, (n - 2 * half + max(stride, 1) - 1) // max(stride, 1)) if n else 1
        depth = np.zeros((cap, h, w), np.float32)
        normals = np.zeros((cap, h, w, 3), np.float32)
        conf = np.zeros((cap, h, w), np.float32)
        refs = np.zeros(cap, np.int32)
        nres = C.c_int32(0)
        self._check(self.fn["estimate_sequence"](self.ctx, views, n, stride, C.byref(cfg), int(filter),
                                                 _ptr(depth), _ptr(normals), _ptr(conf), _ptr(refs),
                                                 cap, C.byref(nres)))
        del keep
        return [FrameResult(int(refs[r]), BundleResult(depth[r], normals[r], conf[r]))
                for r in range(nres.value)]

    def estimate_sequence_multi(self, frames: Sequence[CalibratedView], config: PipelineConfig,
                                devices: Sequence[int], stride: int = 1, filter: Filter = Filter.none,
                                inflight: int = 3, pinned: bool = False) -> list:
        """estimate_sequence sharded over `devices` (contiguous shards, halo
        exchange for the geometric filter; fmvs_estimate_sequence_multi).
        pinned=True hands the library pinned output buffers (direct D2H)."""
        views, keep = _views_c(frames)
        cfg = config.to_c()
        n = len(frames)
        h, w = (frames[0].image.shape if n else (1, 1))
        half = max(config.bundle_size, 1) // 2
        cap = max(1, (n - 2 * half + max(stride, 1) - 1) // max(stride, 1)) if n else 1
        px = h * w
        hbuf = None
        if pinned:
            hbuf = self.fn["host_alloc"](cap * px * 20)
            base = np.ctypeslib.as_array(C.cast(hbuf, C.POINTER(C.c_float)), shape=(cap * px * 5,))
            depth = base[:cap * px].reshape(cap, h, w)
            normals = base[cap * px:4 * cap * px].reshape(cap, h, w, 3)
            conf = base[4 * cap * px:].reshape(cap, h, w)
        else:
            depth = np.zeros((cap, h, w), np.float32)
            normals = np.zeros((cap, h, w, 3), np.float32)
            conf = np.zeros((cap, h, w), np.float32)
        refs = np.zeros(cap, np.int32)
        nres = C.c_int32(0)
        devs = (C.c_int32 * len(devices))(*devices)
        try:
            self._check(self.fn["estimate_sequence_multi"](devs, len(devices), inflight, views, n, stride,
                                                           C.byref(cfg), int(filter), _ptr(depth), _ptr(normals),
                                                           _ptr(conf), _ptr(refs), cap, C.byref(nres)))
            out = [FrameResult(int(refs[r]), BundleResult(depth[r].copy(), normals[r].copy(), conf[r].copy()))
                   for r in range(nres.value)]
        finally:
            if hbuf:
                self.fn["host_free"](hbuf)
        del keep
        return out

    def sequence_plan(self, m: int, shards: int, shard: int, window: int) -> dict:
        """Shard / halo plan of estimate_sequence_multi (host only)."""
        b, e, ni, ne = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        imp = np.zeros(max(m, 1), np.int32)
        exp = np.zeros(max(m, 1), np.int32)
        self._check(self.fn["sequence_plan"](m, shards, shard, window, C.byref(b), C.byref(e), _ptr(imp),
                                             C.byref(ni), _ptr(exp), C.byref(ne)))
        return dict(begin=b.value, end=e.value, imports=imp[:ni.value].tolist(), exports=exp[:ne.value].tolist())

    # ------------------------------------------- output stage (§8f)
    def colorize_depth(self, depth: np.ndarray, lo: float, hi: float) -> np.ndarray:
        """colorize_depth (colorize.hpp:9): uint8 (h, w, 3) viridis."""
        d = _f32(depth)
        h, w = d.shape
        out = np.zeros((h, w, 3), np.uint8)
        self._check(self.fn["colorize_depth"](self.ctx, _ptr(d), w, h, float(lo), float(hi), _ptr(out)))
        return out

    def colorize_normals(self, normals: np.ndarray) -> np.ndarray:
        """colorize_normals (colorize.hpp:12): uint8 (h, w, 3)."""
        n = _f32(normals)
        h, w = n.shape[:2]
        out = np.zeros((h, w, 3), np.uint8)
        self._check(self.fn["colorize_normals"](self.ctx, _ptr(n), w, h, _ptr(out)))
        return out

    def colorize_confidence(self, confidence: np.ndarray) -> np.ndarray:
        """colorize_confidence (colorize.hpp:15): uint8 (h, w, 3) gray."""
        c = _f32(confidence)
        h, w = c.shape
        out = np.zeros((h, w, 3), np.uint8)
        self._check(self.fn["colorize_confidence"](self.ctx, _ptr(c), w, h, _ptr(out)))
        return out

    def write_pfm(self, path: str, data: np.ndarray) -> None:
        """write_pfm (map_io.hpp:25-26): (h, w) -> "Pf", (h, w, 3) -> "PF"."""
        a = _f32(data)
        ch = 1 if a.ndim == 2 else a.shape[2]
        self._check(self.fn["write_pfm"](path.encode(), _ptr(a), a.shape[1], a.shape[0], ch))

    def write_png(self, path: str, rgb: np.ndarray) -> None:
        """write_png (map_io.hpp:27): uint8 (h, w, 3) RGB, byte-identical to the reference."""
        a = np.ascontiguousarray(rgb, np.uint8)
        if a.ndim != 3 or a.shape[2] != 3:
            raise ValueError("write_png: expected an (h, w, 3) uint8 image")
        self._check(self.fn["write_png"](path.encode(), _ptr(a), a.shape[1], a.shape[0]))

    # -------------------------------------- remaining reference helpers
    def gaussian_blur(self, image: np.ndarray, radius: int, sigma: float) -> np.ndarray:
        """gaussian_blur (pipeline.hpp:54): float32 (h, w)."""
        img = np.ascontiguousarray(image, np.uint8)
        h, w = img.shape
        out = np.zeros((h, w), np.float32)
        self._check(self.fn["gaussian_blur"](self.ctx, _ptr(img), w, h, radius, float(sigma), _ptr(out)))
        return out

    def census_transform(self, image: np.ndarray, window_w: int, window_h: int) -> np.ndarray:
        """census_transform (matching.hpp:58): uint64 (h, w)."""
        img = np.ascontiguousarray(image, np.uint8)
        h, w = img.shape
        out = np.zeros((h, w), np.uint64)
        self._check(self.fn["census_transform"](self.ctx, _ptr(img), w, h, window_w, window_h, _ptr(out)))
        return out

    def census_bits_at(self, image: np.ndarray, x: int, y: int, window_w: int, window_h: int) -> int:
        """census_bits_at (matching.hpp:60)."""
        img = np.ascontiguousarray(image, np.uint8)
        h, w = img.shape
        return int(self.fn["census_bits_at"](_ptr(img), w, h, x, y, window_w, window_h))

    def ncc_cost(self, patch_ref, patch_other) -> int:
        """ncc_cost (matching.hpp:64)."""
        a, b = _f32(patch_ref).ravel(), _f32(patch_other).ravel()
        if a.size != b.size:
            raise InvalidInputError("ncc: patches must be non-empty and equal size")
        out = C.c_int32(0)
        self._check(self.fn["ncc_cost"](_ptr(a), _ptr(b), a.size, C.byref(out)))
        return out.value

    def apply_homography(self, hom, x: float, y: float):
        """apply_homography (geometry.hpp:102)."""
        h = np.ascontiguousarray(hom, np.float64).ravel()
        out = np.zeros(2, np.float64)
        self.fn["apply_homography"](_pd(h), float(x), float(y), _pd(out))
        return out

    def cross_ratio(self, p1, p2, p3, p4) -> float:
        """cross_ratio (geometry.hpp:120-123), 2D or 3D points."""
        pts = np.ascontiguousarray([p1, p2, p3, p4], np.float64)
        out = C.c_double(0.0)
        self._check(self.fn["cross_ratio"](_pd(pts), pts.shape[1], C.byref(out)))
        return out.value

    def require_centers_in_front(self, normal, delta_min: float, centers) -> None:
        """require_centers_in_front (geometry.hpp:115-116): GeometryError if violated."""
        n = np.ascontiguousarray(normal, np.float64)
        c = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
        self._check(self.fn["require_centers_in_front"](_pd(n), float(delta_min), _pd(c), len(c)))

    # ------------------------------------------ accuracy scoring (§8f)
    def evaluate(self, est: np.ndarray, gt: np.ndarray, thetas=(1.25, 1.1, 1.05, 1.01)):
        """evaluate (evaluation.hpp:48-49): ({l1_abs, l1_rel, valid_both},
        [{acc, cpl, f, valid_both, valid_est, valid_gt} per theta])."""
        e, g = _f32(est), _f32(gt)
        if e.shape != g.shape or e.size == 0:
            raise InvalidInputError("metrics: maps must be non-empty and equal size")
        h, w = e.shape
        th = np.ascontiguousarray(thetas, np.float64)
        l1 = _abi.L1Result_c()
        sc = (_abi.AccCplF_c * max(1, len(th)))()
        self._check(self.fn["evaluate"](self.ctx, _ptr(e), _ptr(g), w, h, _pd(th), len(th), C.byref(l1), sc))
        keys = ("acc", "cpl", "f", "valid_both", "valid_est", "valid_gt")
        return ({"l1_abs": l1.l1_abs, "l1_rel": l1.l1_rel, "valid_both": int(l1.valid_both)},
                [{k: getattr(sc[i], k) for k in keys} for i in range(len(th))])

    def roc_curve(self, est: np.ndarray, gt: np.ndarray, confidence: np.ndarray, theta: float = 1.05):
        """roc_curve (evaluation.hpp:36-41): (densities[20], error_rates[20])."""
        e, g, c = _f32(est), _f32(gt), _f32(confidence)
        if e.shape != g.shape or e.size == 0:
            raise InvalidInputError("metrics: maps must be non-empty and equal size")
        if c.shape != e.shape:
            raise InvalidInputError("roc: confidence map size differs")
        h, w = e.shape
        dens = np.zeros(20, np.float64)
        errs = np.zeros(20, np.float64)
        self._check(self.fn["roc_curve"](self.ctx, _ptr(e), _ptr(g), _ptr(c), w, h, float(theta),
                                         _pd(dens), _pd(errs)))
        return dens, errs

    # ------------------------------------------------- synthetic scenes
    def render_plane_scene(self, kind: str, width: int, height: int, focal: float, depth: float,
                           views: int, baseline_step: float, seed: int = 1, tilt_deg: float = 0.0,
                           texture_scale: float = 0.5):
        """fronto_scene / slanted_scene + render_scene (render.hpp:41-62).

        Returns (bundle, gt_depth[views,h,w], gt_normals[views,h,w,3])."""
        k = 0 if kind == "fronto" else 1
        px = width * height
        imgs = np.zeros((views, height, width), np.uint8)
        gd = np.zeros((views, height, width), np.float32)
        gn = np.zeros((views, height, width, 3), np.float32)
        intr = (_abi.Intrinsics_c * views)()
        poses = (_abi.Pose_c * views)()
        self._check(self.fn["render_plane_scene"](self.ctx, k, width, height, focal, depth, tilt_deg,
                                                  views, baseline_step, seed, texture_scale,
                                                  _ptr(imgs), _ptr(gd), _ptr(gn), intr, poses))
        bundle = [CalibratedView(imgs[i].copy(), Intrinsics.from_c(intr[i]), Pose.from_c(poses[i]))
                  for i in range(views)]
        del px
        return bundle, gd, gn

    def render_scene(self, scene: "SyntheticScene"):
        """render_scene (render.hpp:41-48) of any SyntheticScene (planes with
        extents, checkerboard or value-noise texture).

        Returns (bundle, gt_depth[views,h,w], gt_normals[views,h,w,3])."""
        n = len(scene.planes)
        planes = (_abi.ScenePlane_c * max(n, 1))()
        for i, sp in enumerate(scene.planes):
            planes[i].point[:] = [float(v) for v in sp.point]
            planes[i].normal[:] = [float(v) for v in sp.normal]
            planes[i].u_axis[:] = [float(v) for v in sp.u_axis]
            planes[i].extent_u = float(sp.extent_u)
            planes[i].extent_v = float(sp.extent_v)
        views = len(scene.poses)
        poses = (_abi.Pose_c * max(views, 1))(*[p.to_c() for p in scene.poses])
        k = scene.intrinsics
        h, w = max(k.height, 0), max(k.width, 0)
        imgs = np.zeros((views, h, w), np.uint8)
        gd = np.zeros((views, h, w), np.float32)
        gn = np.zeros((views, h, w, 3), np.float32)
        intr = k.to_c()
        self._check(self.fn["render_scene"](self.ctx, planes, n, poses, views, C.byref(intr),
                                            int(scene.texture), float(scene.texture_scale),
                                            int(scene.seed), _ptr(imgs), _ptr(gd), _ptr(gn)))
        bundle = [CalibratedView(imgs[i].copy(), k, scene.poses[i]) for i in range(views)]
        return bundle, gd, gn


class TextureKind(enum.IntEnum):  # render.hpp:12
    Checkerboard = 0
    ValueNoise = 1


@dataclass
class ScenePlane:  # render.hpp:16-22
    point: Sequence[float] = (0.0, 0.0, 0.0)
    normal: Sequence[float] = (0.0, 0.0, -1.0)
    u_axis: Sequence[float] = (1.0, 0.0, 0.0)
    extent_u: float = float("inf")
    extent_v: float = float("inf")


@dataclass
class SyntheticScene:  # render.hpp:24-31
    planes: list
    poses: list
    intrinsics: "Intrinsics"
    texture: TextureKind = TextureKind.ValueNoise
    texture_scale: float = 0.5
    seed: int = 1


def lateral_trajectory(views: int, step: float) -> list:
    """lateral_trajectory (render.cpp:143-148)."""
    return [Pose(np.eye(3), np.array([(i - (views - 1) / 2.0) * step, 0.0, 0.0])) for i in range(views)]


def default_backend() -> Backend:
    return Backend.b200()


def estimate_bundle(bundle: Sequence[CalibratedView], config: PipelineConfig) -> BundleResult:
    """Module-level drop-in for fassmvs::estimate_bundle on the B200 library."""
    return default_backend().estimate_bundle(bundle, config)
