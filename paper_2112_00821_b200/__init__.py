"""B200-native FaSS-MVS per-frame depth/normal/confidence pipeline.

The product is ``_lib/libfmvs.so``: hand-written sm_100a CUDA kernels and a
C++ host driver behind the C ABI in ``include/fmvs.h``. This package is the
Python binding of that ABI, mirroring the reference API names
(``fassmvs::estimate_bundle`` etc.). There is no CPU fallback: importing the
binding when the library is not built raises.
"""
from .fassmvs import (  # noqa: F401
    AggregatedVolume, Backend, BundleResult, CalibratedView, ConfigError, ConsistencyView,
    CostFunctionSpec, CostKind, CostVolume, CudaError, DepthLookup, Filter, FrameResult,
    GeomFilterConfig, GeometryError, Intrinsics, InvalidInputError, PipelineConfig, PlaneStack,
    Pose, RangeKind, RangePolicy, ScenePlane, SgmConfig, SgmVariant, SyntheticScene, TextureKind,
    default_backend, estimate_bundle, lateral_trajectory)

__all__ = [
    "AggregatedVolume", "Backend", "BundleResult", "CalibratedView", "ConfigError",
    "ConsistencyView", "CostFunctionSpec", "CostKind", "CostVolume", "CudaError", "DepthLookup",
    "Filter", "FrameResult", "GeomFilterConfig", "GeometryError", "Intrinsics",
    "InvalidInputError", "PipelineConfig", "PlaneStack", "Pose", "RangeKind", "RangePolicy",
    "ScenePlane", "SgmConfig", "SgmVariant", "SyntheticScene", "TextureKind", "default_backend",
    "estimate_bundle", "lateral_trajectory",
]
