"""ctypes mirror of include/fmvs.h (the C ABI of the B200 library).

The same declarations bind any library exporting the fmvs_* entry points
under a name prefix; the parity tests use that to drive the reference oracle
(oracle/_ref, prefix ``ref_``) through the identical Python API.
"""
from __future__ import annotations

import ctypes as C

FMVS_OK = 0
FMVS_ERR_INVALID_INPUT = 1
FMVS_ERR_CONFIG = 2
FMVS_ERR_GEOMETRY = 3
FMVS_ERR_CUDA = 4
FMVS_ERR_CAPACITY = 5


class Intrinsics_c(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class Pose_c(C.Structure):
    _fields_ = [("rotation", C.c_double * 9), ("center", C.c_double * 3)]


class ScenePlane_c(C.Structure):
    _fields_ = [("point", C.c_double * 3), ("normal", C.c_double * 3), ("u_axis", C.c_double * 3),
                ("extent_u", C.c_double), ("extent_v", C.c_double)]


class View_c(C.Structure):
    _fields_ = [("image", C.c_void_p), ("intrinsics", Intrinsics_c), ("pose", Pose_c)]


class PlaneStack_c(C.Structure):
    _fields_ = [("normal", C.c_double * 3), ("distances", C.c_void_p), ("count", C.c_int32)]


class SgmConfig_c(C.Structure):
    _fields_ = [("variant", C.c_int32), ("paths", C.c_int32), ("phi1", C.c_double),
                ("phi2_adaptive", C.c_int32), ("phi2_fixed", C.c_double), ("alpha", C.c_double),
                ("beta", C.c_double), ("penalty_scale", C.c_int32)]


class CostSpec_c(C.Structure):
    _fields_ = [("kind", C.c_int32), ("window_w", C.c_int32), ("window_h", C.c_int32)]


class Config_c(C.Structure):
    _fields_ = [("bundle_size", C.c_int32), ("pyramid_levels", C.c_int32), ("d_min", C.c_double),
                ("d_max", C.c_double), ("sweep_normal", C.c_double * 3), ("range_kind", C.c_int32),
                ("range_value", C.c_double), ("max_planes", C.c_int32), ("sgm", SgmConfig_c),
                ("cost", CostSpec_c), ("normal_smoothing_radius", C.c_int32)]


class ConsistencyView_c(C.Structure):
    _fields_ = [("depth", C.c_void_p), ("width", C.c_int32), ("height", C.c_int32),
                ("intrinsics", Intrinsics_c), ("pose", Pose_c)]


class GeomFilterConfig_c(C.Structure):
    _fields_ = [("eta_r", C.c_double), ("eta_h", C.c_int32), ("lookup", C.c_int32)]


class L1Result_c(C.Structure):
    _fields_ = [("l1_abs", C.c_double), ("l1_rel", C.c_double), ("valid_both", C.c_uint64)]


class AccCplF_c(C.Structure):
    _fields_ = [("acc", C.c_double), ("cpl", C.c_double), ("f", C.c_double), ("valid_both", C.c_uint64),
                ("valid_est", C.c_uint64), ("valid_gt", C.c_uint64)]


class LevelStats_c(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("planes", C.c_int32),
                ("entries", C.c_uint64)]


P = C.c_void_p
I32 = C.c_int32
U64 = C.c_uint64
D = C.c_double
PD = C.POINTER(C.c_double)

# name -> (restype, argtypes); names without the prefix.
SIGNATURES = {
    "abi_version": (I32, []),
    "last_error": (C.c_char_p, []),
    "config_default": (None, [C.POINTER(Config_c), D, D]),
    "ctx_create": (C.c_int, [I32, C.POINTER(P)]),
    "ctx_destroy": (None, [P]),
    "ctx_synchronize": (C.c_int, [P]),
    "ctx_level_stats": (I32, [P, C.POINTER(LevelStats_c), I32]),
    "ctx_last_launch_count": (C.c_int64, [P]),
    "ctx_stream": (P, [P]),
    "ctx_set_timing": (None, [P, I32]),
    "ctx_stage_count": (I32, [P]),
    "ctx_stage_name": (C.c_char_p, [P, I32]),
    "ctx_stage_time": (C.c_int, [P, I32, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "ctx_stage_reset": (None, [P]),
    "ctx_sweep_stats": (C.c_int, [P, C.POINTER(C.c_uint64)]),
    "ctx_set_capture": (C.c_int, [P, I32]),
    "ctx_capture_sizes": (C.c_int, [P, C.POINTER(I32), C.POINTER(I32), C.POINTER(U64)]),
    "ctx_capture_copy": (C.c_int, [P, P, P, P, P, P, P, P]),
    "host_alloc": (P, [U64]),
    "host_free": (None, [P]),
    "estimate_bundle": (C.c_int, [P, C.POINTER(View_c), I32, C.POINTER(Config_c), P, P, P]),
    "estimate_bundle_device": (C.c_int, [P, C.POINTER(View_c), I32, C.POINTER(Config_c), P, P, P]),
    "plane_homography": (C.c_int, [PD, D, C.POINTER(Intrinsics_c), C.POINTER(Pose_c),
                                   C.POINTER(Intrinsics_c), C.POINTER(Pose_c), PD]),
    "bounding_distances": (C.c_int, [D, D, PD, C.POINTER(Intrinsics_c), PD, PD]),
    "plane_distances": (C.c_int, [C.POINTER(Intrinsics_c), C.POINTER(Pose_c), C.POINTER(Intrinsics_c),
                                  C.POINTER(Pose_c), D, D, PD, I32, PD, I32, C.POINTER(I32)]),
    "depth_from_plane": (D, [D, D, PD, D, C.POINTER(Intrinsics_c)]),
    "adaptive_phi2": (D, [D, D, D, D]),
    "parabola_refine": (C.c_int, [D, D, D, D, D, D, PD]),
    "build_pyramids": (C.c_int, [P, C.POINTER(View_c), I32, I32, P, U64, C.POINTER(Intrinsics_c)]),
    "refine_range": (C.c_int, [P, P, I32, I32, I32, D, D, D, C.POINTER(PlaneStack_c),
                               C.POINTER(Intrinsics_c), P, P]),
    "sweep_cost_volume": (C.c_int, [P, C.POINTER(View_c), I32, I32, C.POINTER(PlaneStack_c), P, P,
                                    C.POINTER(CostSpec_c), P, P, P, P, U64, C.POINTER(U64),
                                    C.POINTER(I32)]),
    "compute_normal_offsets": (C.c_int, [P, P, P, I32, I32, C.POINTER(PlaneStack_c),
                                         C.POINTER(Intrinsics_c), P]),
    "aggregate": (C.c_int, [P, I32, I32, C.POINTER(PlaneStack_c), P, P, P, P, U64, P,
                            C.POINTER(SgmConfig_c), C.POINTER(Intrinsics_c), P, P, I32, I32, P]),
    "aggregate_single_path": (C.c_int, [P, I32, I32, C.POINTER(PlaneStack_c), P, P, P, P, U64, P,
                                        C.POINTER(SgmConfig_c), C.POINTER(Intrinsics_c), P, P, I32, I32,
                                        P]),
    "wta": (C.c_int, [P, I32, I32, P, P, P, P, U64, P]),
    "median_filter_5x5": (C.c_int, [P, P, I32, I32, P]),
    "normals_from_depth": (C.c_int, [P, P, I32, I32, C.POINTER(Intrinsics_c), P]),
    "smooth_normals": (C.c_int, [P, P, P, I32, I32, I32, P]),
    "confidence_map": (C.c_int, [P, P, I32, I32, PD, D, P]),
    "upscale_nearest": (C.c_int, [P, P, I32, I32, I32, I32, I32, P]),
    "render_plane_scene": (C.c_int, [P, I32, I32, I32, D, D, D, I32, D, U64, D, P, P, P,
                                     C.POINTER(Intrinsics_c), C.POINTER(Pose_c)]),
    "render_scene": (C.c_int, [P, C.POINTER(ScenePlane_c), I32, C.POINTER(Pose_c), I32,
                               C.POINTER(Intrinsics_c), I32, D, U64, P, P, P]),
    "dog_mask": (C.c_int, [P, P, I32, I32, P]),
    "apply_mask": (C.c_int, [P, P, P, P, I32, I32, P]),
    "geom_filter_config_default": (None, [C.POINTER(GeomFilterConfig_c)]),
    "geometric_consistency_mask": (C.c_int, [P, C.POINTER(ConsistencyView_c), I32, I32,
                                             C.POINTER(GeomFilterConfig_c), P]),
    "estimate_sequence": (C.c_int, [P, C.POINTER(View_c), I32, I32, C.POINTER(Config_c), I32, P, P,
                                    P, P, I32, C.POINTER(I32)]),
    "estimate_sequence_multi": (C.c_int, [C.POINTER(I32), I32, I32, C.POINTER(View_c), I32, I32,
                                          C.POINTER(Config_c), I32, P, P, P, P, I32, C.POINTER(I32)]),
    "sequence_plan": (C.c_int, [I32, I32, I32, I32, C.POINTER(I32), C.POINTER(I32), P, C.POINTER(I32), P,
                                C.POINTER(I32)]),
    "colorize_depth": (C.c_int, [P, P, I32, I32, D, D, P]),
    "colorize_normals": (C.c_int, [P, P, I32, I32, P]),
    "colorize_confidence": (C.c_int, [P, P, I32, I32, P]),
    "write_pfm": (C.c_int, [C.c_char_p, P, I32, I32, I32]),
    "write_png": (C.c_int, [C.c_char_p, P, I32, I32]),
    "evaluate": (C.c_int, [P, P, P, I32, I32, PD, I32, C.POINTER(L1Result_c), C.POINTER(AccCplF_c)]),
    "roc_curve": (C.c_int, [P, P, P, P, I32, I32, D, PD, PD]),
    "gaussian_blur": (C.c_int, [P, P, I32, I32, I32, D, P]),
    "census_transform": (C.c_int, [P, P, I32, I32, I32, I32, P]),
    "census_bits_at": (U64, [P, I32, I32, I32, I32, I32, I32]),
    "ncc_cost": (C.c_int, [P, P, I32, C.POINTER(I32)]),
    "apply_homography": (None, [PD, D, D, PD]),
    "cross_ratio": (C.c_int, [PD, I32, PD]),
    "require_centers_in_front": (C.c_int, [PD, D, PD, I32]),
}

# Entry points only the oracle library has.
ORACLE_EXTRAS = {
    "worker_count": (C.c_int, []),
}


def bind(lib: C.CDLL, prefix: str, extras: dict | None = None) -> dict:
    """Returns {name: ctypes function} for every declared entry point present."""
    table = dict(SIGNATURES)
    if extras:
        table.update(extras)
    out = {}
    for name, (res, args) in table.items():
        fn = getattr(lib, prefix + name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
        out[name] = fn
    return out
