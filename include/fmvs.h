/*
 * fmvs.h — C ABI of the B200-native FaSS-MVS per-frame depth/normal path.
 *
 * This is the drop-in boundary for the reference's C++ API in
 * /root/reference/proj/include/fassmvs/ (SURVEY.md §8b). Plain C types only:
 * pointers, sizes, POD structs. Every entry point cites the reference
 * interface it replaces. Host code above this ABI (the C++ adapter
 * include/fassmvs_b200.hpp, the Python binding paper_2112_00821_b200/) maps
 * return codes back to the reference's exception types (errors.hpp:10-24).
 *
 * Conventions
 *   - images are 8-bit grayscale, row-major, width*height bytes
 *     (ImageU8 = Raster<uint8_t>, raster.hpp:13-58)
 *   - float maps are row-major width*height (DepthMap/ConfidenceMap,
 *     raster.hpp:60-61); normal maps are interleaved xyz, 3*width*height
 *     floats (NormalMap = Raster<Eigen::Vector3f>, raster.hpp:62)
 *   - 3x3 matrices are row-major double[9]
 *   - return code: FMVS_OK or one of the FMVS_ERR_* codes; the message of the
 *     last failure on the calling thread is fmvs_last_error()
 *   - a context owns one CUDA stream and its device arenas; it is not
 *     reentrant, distinct contexts are fully concurrent (README.md:160-162)
 */
#ifndef FMVS_H
#define FMVS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMVS_ABI_VERSION 1

/* Return codes. 1..3 mirror the reference exception types (errors.hpp:10-24)
 * whose CLI exit codes are 1/2/1 (tools/fassmvs.cpp:338-353). */
enum {
    FMVS_OK = 0,
    FMVS_ERR_INVALID_INPUT = 1, /* fassmvs::InvalidInputError */
    FMVS_ERR_CONFIG = 2,        /* fassmvs::ConfigError */
    FMVS_ERR_GEOMETRY = 3,      /* fassmvs::GeometryError */
    FMVS_ERR_CUDA = 4,          /* CUDA runtime / device failure (no reference analogue) */
    FMVS_ERR_CAPACITY = 5       /* caller-provided output buffer too small */
};

/* Intrinsics (geometry.hpp:19-39). */
typedef struct fmvs_intrinsics {
    double fx, fy, cx, cy;
    int32_t width, height;
} fmvs_intrinsics;

/* Pose (geometry.hpp:44-55): rotation maps reference-frame vectors into the
 * camera frame (row-major), center in the reference frame. */
typedef struct fmvs_pose {
    double rotation[9];
    double center[3];
} fmvs_pose;

/* CalibratedView (geometry.hpp:57-63). */
typedef struct fmvs_view {
    const uint8_t* image; /* width*height bytes, row-major */
    fmvs_intrinsics intrinsics;
    fmvs_pose pose;
} fmvs_view;

/* PlaneStack (geometry.hpp:75-94): shared normal + strictly decreasing
 * distances. */
typedef struct fmvs_plane_stack {
    double normal[3];
    const double* distances;
    int32_t count;
} fmvs_plane_stack;

enum { FMVS_COST_CENSUS = 0, FMVS_COST_NCC = 1 };              /* CostKind, matching.hpp:12 */
enum { FMVS_SGM_PLANE = 0, FMVS_SGM_SURFACE_NORMAL = 1,
       FMVS_SGM_PATH_GRADIENT = 2 };                            /* SgmVariant, sgm.hpp:13-17 */
enum { FMVS_RANGE_FULL = 0, FMVS_RANGE_FIXED = 1,
       FMVS_RANGE_SPACING_MULTIPLE = 2 };                       /* RangePolicy::Kind, pipeline.hpp:13-18 */

/* SgmConfig (sgm.hpp:19-32). */
typedef struct fmvs_sgm_config {
    int32_t variant;
    int32_t paths; /* 8 or 4 */
    double phi1;
    int32_t phi2_adaptive;
    double phi2_fixed;
    double alpha;
    double beta;
    int32_t penalty_scale;
} fmvs_sgm_config;

/* CostFunctionSpec (matching.hpp:14-23). */
typedef struct fmvs_cost_spec {
    int32_t kind;
    int32_t window_w;
    int32_t window_h;
} fmvs_cost_spec;

/* PipelineConfig (pipeline.hpp:22-35) incl. DepthBounds and RangePolicy. */
typedef struct fmvs_config {
    int32_t bundle_size;
    int32_t pyramid_levels;
    double d_min, d_max;
    double sweep_normal[3];
    int32_t range_kind;
    double range_value;
    int32_t max_planes;
    fmvs_sgm_config sgm;
    fmvs_cost_spec cost;
    int32_t normal_smoothing_radius;
} fmvs_config;

/* Per-level statistics of the last estimate on a context. */
typedef struct fmvs_level_stats {
    int32_t width, height;
    int32_t planes;        /* global plane-stack size of the level */
    uint64_t entries;      /* sum over pixels of CostVolume::count */
} fmvs_level_stats;

typedef struct fmvs_ctx fmvs_ctx;

/* ---------------------------------------------------------------- misc -- */
int32_t fmvs_abi_version(void);
const char* fmvs_last_error(void);
/* Fills the reference defaults (PipelineConfig ctor, pipeline.hpp:22-35;
 * SgmConfig sgm.hpp:19-32; CostFunctionSpec matching.hpp:14-23). */
void fmvs_config_default(fmvs_config* cfg, double d_min, double d_max);

/* ------------------------------------------------------------- context -- */
/* A context owns one CUDA stream and the device arenas of one GPU; device
 * < 0 selects the calling thread's current CUDA device. */
int fmvs_ctx_create(int32_t device, fmvs_ctx** out);
/* The calling thread's current CUDA device (cudaGetDevice), -1 on failure. */
int32_t fmvs_current_device(void);
void fmvs_ctx_destroy(fmvs_ctx* ctx);
int fmvs_ctx_synchronize(fmvs_ctx* ctx);
/* Per-level statistics of the last estimate_bundle on this context; returns
 * the number of levels written (<= capacity). */
int32_t fmvs_ctx_level_stats(fmvs_ctx* ctx, fmvs_level_stats* out, int32_t capacity);
/* Number of kernels the last estimate enqueued. */
int64_t fmvs_ctx_last_launch_count(fmvs_ctx* ctx);
/* The context's CUDA stream (cudaStream_t), for event timing by callers. */
void* fmvs_ctx_stream(fmvs_ctx* ctx);
/* Optional per-stage CUDA-event timing on the context stream (stage times
 * accumulate over calls until fmvs_ctx_stage_reset). */
void fmvs_ctx_set_timing(fmvs_ctx* ctx, int32_t enable);
int32_t fmvs_ctx_stage_count(fmvs_ctx* ctx);
const char* fmvs_ctx_stage_name(fmvs_ctx* ctx, int32_t index);
int fmvs_ctx_stage_time(fmvs_ctx* ctx, int32_t index, double* ms, int64_t* calls);
void fmvs_ctx_stage_reset(fmvs_ctx* ctx);
/* Diagnostics of the certified census sweep (enabled by FMVS_SWEEP_STATS=1 at
 * context creation): {hypothesis-view evaluations, evaluations with an
 * undecided bit, undecided bits, exact-path views, tile-plane iterations run,
 * tile-plane iterations skipped, exact samples taken, 0}; read-and-clear. */
int fmvs_ctx_sweep_stats(fmvs_ctx* ctx, uint64_t out[8]);
/* Stage capture (parity debugging, tests/test_fullsize_gpu.py): when a level
 * >= 0 is set, the next estimate_bundle on this context keeps that level's
 * ragged layout (the reference's CostVolume first/count/offset), u16 costs,
 * u32 SGM aggregate, WTA winners and pre-median depth in host memory (one
 * extra stream synchronisation). -1 disables. Sizes first, then copy into
 * caller buffers of width*height (first, count, offset, winners, depth_raw)
 * and `entries` (costs, aggregate) elements. */
int fmvs_ctx_set_capture(fmvs_ctx* ctx, int32_t level);
int fmvs_ctx_capture_sizes(fmvs_ctx* ctx, int32_t* width, int32_t* height, uint64_t* entries);
int fmvs_ctx_capture_copy(fmvs_ctx* ctx, int32_t* first, int32_t* count, uint64_t* offset,
                          uint16_t* costs, uint32_t* aggregate, int32_t* winners,
                          float* depth_raw);
/* Pinned host memory for zero-staging H2D/D2H of bundles and maps. */
void* fmvs_host_alloc(uint64_t bytes);
void fmvs_host_free(void* ptr);

/* ------------------------------------------------------------ hot path -- */
/* fassmvs::estimate_bundle (pipeline.hpp:79-80, pipeline.cpp:200-309).
 * Host buffers in and out: depth/confidence width*height floats, normals
 * 3*width*height floats, all at the reference view's full resolution.
 * Blocking: returns when the outputs are written. */
int fmvs_estimate_bundle(fmvs_ctx* ctx, const fmvs_view* views, int32_t n_views,
                         const fmvs_config* cfg, float* depth, float* normals_xyz,
                         float* confidence);

/* Device-resident variant: views[k].image are DEVICE pointers, outputs are
 * DEVICE pointers; enqueued on the context stream and returns without
 * waiting (fmvs_ctx_synchronize to wait). Same validation and results. */
int fmvs_estimate_bundle_device(fmvs_ctx* ctx, const fmvs_view* views, int32_t n_views,
                                const fmvs_config* cfg, float* d_depth, float* d_normals_xyz,
                                float* d_confidence);

/* ------------------------------------------------- host-side geometry -- */
/* plane_homography (geometry.hpp:100-103, geometry.cpp:100-114). */
int fmvs_plane_homography(const double normal[3], double distance,
                          const fmvs_intrinsics* ref_intr, const fmvs_pose* ref_pose,
                          const fmvs_intrinsics* other_intr, const fmvs_pose* other_pose,
                          double out_h[9]);
/* bounding_distances (geometry.hpp:110-112, geometry.cpp:121-145). */
int fmvs_bounding_distances(double d_min, double d_max, const double normal[3],
                            const fmvs_intrinsics* ref_intr, double* delta_min,
                            double* delta_max);
/* plane_distances (geometry.hpp:132-135, geometry.cpp:183-297). Writes at
 * most capacity distances; *count receives the full count
 * (FMVS_ERR_CAPACITY when it exceeds capacity). */
int fmvs_plane_distances(const fmvs_intrinsics* ref_intr, const fmvs_pose* ref_pose,
                         const fmvs_intrinsics* other_intr, const fmvs_pose* other_pose,
                         double delta_min, double delta_max, const double normal[3],
                         int32_t max_planes, double* out, int32_t capacity, int32_t* count);
/* depth_from_plane (geometry.hpp:140, geometry.cpp:299-306). */
double fmvs_depth_from_plane(double x, double y, const double normal[3], double distance,
                             const fmvs_intrinsics* intr);
/* adaptive_phi2 (sgm.hpp:36, sgm.cpp:22-24). */
double fmvs_adaptive_phi2(double phi1, double alpha, double beta, double intensity_delta);
/* parabola_refine (sgm.hpp:98-101, sgm.cpp:351-363). */
int fmvs_parabola_refine(double d_prev, double d_win, double d_next, double c_prev,
                         double c_win, double c_next, double* out);

/* -------------------------------------------- device stages (host I/O) -- */
/* build_pyramids (pipeline.hpp:50, pipeline.cpp:79-126): out_images holds
 * levels x n_views images back to back (level-major, each level's size from
 * out_intr[level*n_views + k]); capacity in bytes. */
int fmvs_build_pyramids(fmvs_ctx* ctx, const fmvs_view* views, int32_t n_views,
                        int32_t levels, uint8_t* out_images, uint64_t capacity,
                        fmvs_intrinsics* out_intr);

/* refine_range (pipeline.hpp:63-65, pipeline.cpp:136-173). coarser and intr
 * may be NULL (required by the spacing policy). */
int fmvs_refine_range(fmvs_ctx* ctx, const float* prior, int32_t width, int32_t height,
                      int32_t range_kind, double range_value, double d_min, double d_max,
                      const fmvs_plane_stack* coarser, const fmvs_intrinsics* intr, float* lo,
                      float* hi);

/* sweep_cost_volume (matching.hpp:74-76, matching.cpp:116-294). Outputs the
 * dynamic CostVolume (matching.hpp:36-53): first/count/offset per pixel and
 * costs (capacity entries; *total receives the entry count, FMVS_ERR_CAPACITY
 * when it exceeds capacity). */
int fmvs_sweep_cost_volume(fmvs_ctx* ctx, const fmvs_view* views, int32_t n_views,
                           int32_t ref_index, const fmvs_plane_stack* planes, const float* lo,
                           const float* hi, const fmvs_cost_spec* cost, int32_t* first,
                           int32_t* count, uint64_t* offset, uint16_t* costs, uint64_t capacity,
                           uint64_t* total, int32_t* per_side);

/* compute_normal_offsets (sgm.hpp:66-68, sgm.cpp:252-299): out holds 4
 * int16 shifts per pixel (canonical dirs, sgm.hpp:55-56). */
int fmvs_compute_normal_offsets(fmvs_ctx* ctx, const float* prior_normals_xyz,
                                const float* prior_depth, int32_t width, int32_t height,
                                const fmvs_plane_stack* planes, const fmvs_intrinsics* intr,
                                int16_t* out);

/* aggregate / aggregate_single_path (sgm.hpp:86-96, sgm.cpp:301-331). The
 * volume is given as the reference's ragged layout. dir_x = dir_y = 0 runs
 * all cfg->paths directions; otherwise the single path (dir_x, dir_y).
 * prior_* may be NULL unless the variant is SurfaceNormal. */
int fmvs_aggregate(fmvs_ctx* ctx, int32_t width, int32_t height, const fmvs_plane_stack* planes,
                   const int32_t* first, const int32_t* count, const uint64_t* offset,
                   const uint16_t* costs, uint64_t total, const uint8_t* image,
                   const fmvs_sgm_config* cfg, const fmvs_intrinsics* intr,
                   const float* prior_normals_xyz, const float* prior_depth, int32_t dir_x,
                   int32_t dir_y, uint32_t* out_values);
/* aggregate_single_path (sgm.hpp:91-95, sgm.cpp:301-315) for any integer step
 * (dir_x, dir_y), including non-unit steps and (0, 0) (no lines: zeros). */
int fmvs_aggregate_single_path(fmvs_ctx* ctx, int32_t width, int32_t height,
                               const fmvs_plane_stack* planes, const int32_t* first,
                               const int32_t* count, const uint64_t* offset, const uint16_t* costs,
                               uint64_t total, const uint8_t* image, const fmvs_sgm_config* cfg,
                               const fmvs_intrinsics* intr, const float* prior_normals_xyz,
                               const float* prior_depth, int32_t dir_x, int32_t dir_y,
                               uint32_t* out_values);

/* wta (sgm.hpp:93, sgm.cpp:333-349). */
int fmvs_wta(fmvs_ctx* ctx, int32_t width, int32_t height, const int32_t* first,
             const int32_t* count, const uint64_t* offset, const uint32_t* values,
             uint64_t total, int32_t* winners);

/* median_filter_5x5 (pipeline.hpp:70, pipeline.cpp:175-198). */
int fmvs_median_filter_5x5(fmvs_ctx* ctx, const float* depth, int32_t width, int32_t height,
                           float* out);

/* normals_from_depth / smooth_normals / confidence_map (surface.hpp:11-24,
 * surface.cpp:9-104). */
int fmvs_normals_from_depth(fmvs_ctx* ctx, const float* depth, int32_t width, int32_t height,
                            const fmvs_intrinsics* intr, float* out_xyz);
int fmvs_smooth_normals(fmvs_ctx* ctx, const float* raw_xyz, const uint8_t* image,
                        int32_t width, int32_t height, int32_t radius, float* out_xyz);
int fmvs_confidence_map(fmvs_ctx* ctx, const float* normals_xyz, int32_t width, int32_t height,
                        const double sweep_normal[3], double rho_degrees, float* out);

/* upscale_nearest (pipeline.hpp:58-59, pipeline.cpp:91-134); channels = 1
 * (DepthMap) or 3 (NormalMap). */
int fmvs_upscale_nearest(fmvs_ctx* ctx, const float* in, int32_t in_width, int32_t in_height,
                         int32_t channels, int32_t out_width, int32_t out_height, float* out);

/* --------------------------------------------- synthetic input (bench) -- */
/* render_scene over fronto_scene / slanted_scene (render.hpp:41-62,
 * render.cpp:52-183) on the device: kind 0 = fronto, 1 = slanted. images:
 * n_views*width*height bytes; gt_depth / gt_normals_xyz of every view (may be
 * NULL); intr / poses receive the cameras. */
int fmvs_render_plane_scene(fmvs_ctx* ctx, int32_t kind, int32_t width, int32_t height,
                            double focal, double depth, double tilt_deg, int32_t n_views,
                            double baseline_step, uint64_t seed, double texture_scale,
                            uint8_t* images, float* gt_depth, float* gt_normals_xyz,
                            fmvs_intrinsics* intr, fmvs_pose* poses);

/* render_scene (render.hpp:12-48, render.cpp:52-141) on the device for any
 * SyntheticScene: planes (ScenePlane: point, normal, u_axis, half extents;
 * +inf = unbounded), one view per pose, texture 0 = checkerboard, 1 = value
 * noise. Each pixel's ray takes the nearest plane hit inside its extents;
 * outputs as fmvs_render_plane_scene (images n_poses*width*height bytes;
 * gt_depth / gt_normals_xyz may be NULL). Errors as the reference:
 * intrinsics, empty planes/poses, texture scale, then each pose in order. */
typedef struct fmvs_scene_plane {
    double point[3], normal[3], u_axis[3];
    double extent_u, extent_v;
} fmvs_scene_plane;
#define FMVS_TEXTURE_CHECKERBOARD 0
#define FMVS_TEXTURE_VALUE_NOISE 1
int fmvs_render_scene(fmvs_ctx* ctx, const fmvs_scene_plane* planes, int32_t n_planes,
                      const fmvs_pose* poses, int32_t n_poses, const fmvs_intrinsics* intrinsics,
                      int32_t texture, double texture_scale, uint64_t seed, uint8_t* images,
                      float* gt_depth, float* gt_normals_xyz);

/* ------------------------------------------ post-filters -- */
/* dog_mask (postfilter.hpp:13-18, postfilter.cpp:67-79): out = width*height
 * bytes, 1 = textured (keep). */
int fmvs_dog_mask(fmvs_ctx* ctx, const uint8_t* image, int32_t width, int32_t height,
                  uint8_t* out);
/* apply_mask (postfilter.hpp:20-22, postfilter.cpp:81-93), in place on host
 * maps of width*height pixels (normals interleaved xyz). */
int fmvs_apply_mask(fmvs_ctx* ctx, float* depth, float* normals_xyz, float* confidence,
                    int32_t width, int32_t height, const uint8_t* mask);
/* ConsistencyView (postfilter.hpp:24-28): depth map (width*height floats) with
 * its camera. */
typedef struct fmvs_consistency_view {
    const float* depth;
    int32_t width, height;
    fmvs_intrinsics intrinsics;
    fmvs_pose pose;
} fmvs_consistency_view;
enum { FMVS_LOOKUP_NEAREST = 0, FMVS_LOOKUP_BILINEAR = 1 };   /* DepthLookup, postfilter.hpp:30 */
/* GeomFilterConfig (postfilter.hpp:32-36). */
typedef struct fmvs_geom_filter_config {
    double eta_r;   /* reprojection threshold, pixels (10) */
    int32_t eta_h;  /* required consistent neighbour views (3) */
    int32_t lookup; /* FMVS_LOOKUP_* (nearest) */
} fmvs_geom_filter_config;
void fmvs_geom_filter_config_default(fmvs_geom_filter_config* cfg);
/* geometric_consistency_mask (postfilter.hpp:44-45, postfilter.cpp:95-160):
 * keep = width*height bytes of window[ref_index]; 1 = keep. */
int fmvs_geometric_consistency_mask(fmvs_ctx* ctx, const fmvs_consistency_view* window,
                                    int32_t n_views, int32_t ref_index,
                                    const fmvs_geom_filter_config* cfg, uint8_t* keep);

/* -------------------------------------- sequence driver -- */
enum { FMVS_FILTER_NONE = 0, FMVS_FILTER_DOG = 1, FMVS_FILTER_GEOM = 2, FMVS_FILTER_BOTH = 3 };
/* The `fassmvs estimate` loop over a frame sequence (tools/fassmvs.cpp:
 * 92-176) without the file I/O: bundles of cfg->bundle_size consecutive
 * frames centred on ref = half, half + stride, ... while ref + half <
 * n_frames, each estimated on the device; then (filter) the DoG texture mask
 * of each result's reference frame, and the geometric consistency mask of each
 * result against a window of min(5, m) neighbouring results (all masks
 * computed before any is applied, :163-176). Frames are host images; results
 * are written result-major: depth[r*W*H], normals_xyz[r*3*W*H],
 * confidence[r*W*H] (all frames must share one size), ref_frames[r] = the
 * reference frame index. *n_results is always set; FMVS_ERR_CAPACITY if it
 * exceeds capacity. Errors follow the CLI: ConfigError for an invalid bundle
 * size, stride or filter and for a geometric window smaller than eta_h + 1;
 * InvalidInputError for a sequence shorter than one bundle. */
int fmvs_estimate_sequence(fmvs_ctx* ctx, const fmvs_view* frames, int32_t n_frames,
                           int32_t stride, const fmvs_config* cfg, int32_t filter,
                           float* depth, float* normals_xyz, float* confidence,
                           int32_t* ref_frames, int32_t capacity, int32_t* n_results);

/* The same loop sharded over GPUs: devices[0..n_devices) own
 * contiguous shards of the result list (a device id may repeat: several
 * shards on one GPU), each run by one host thread with `inflight` bundles in
 * flight (one stream each) and a post stream for the filters. Results stream
 * back as soon as they are final (direct async D2H when the three output
 * buffers are pinned, e.g. fmvs_host_alloc; else through pinned staging),
 * device memory is a bounded pool of result slots, and the geometric filter's
 * window crosses shard boundaries through a halo of DoG-filtered depth maps
 * copied peer to peer (cudaMemcpyPeerAsync over NVLink, after the producer's
 * event). Arguments, outputs and errors as fmvs_estimate_sequence, whose
 * results it reproduces bit for bit for any device list. */
int fmvs_estimate_sequence_multi(const int32_t* devices, int32_t n_devices, int32_t inflight,
                                 const fmvs_view* frames, int32_t n_frames, int32_t stride,
                                 const fmvs_config* cfg, int32_t filter, float* depth,
                                 float* normals_xyz, float* confidence, int32_t* ref_frames,
                                 int32_t capacity, int32_t* n_results);

/* Shard and halo plan of fmvs_estimate_sequence_multi (host only, no GPU):
 * for m results over n_shards contiguous shards and a geometric window of
 * `window` results (min(5, m) with the geometric filter, else 0), shard
 * `shard`'s result range [*begin, *end), the results it imports from other
 * shards and the results it exports to them (ascending; arrays of m entries
 * or NULL). */
int fmvs_sequence_plan(int32_t m, int32_t n_shards, int32_t shard, int32_t window, int32_t* begin,
                       int32_t* end, int32_t* imports, int32_t* n_imports, int32_t* exports,
                       int32_t* n_exports);

/* ------------------------------------- output stage -- */
/* colorize_depth / colorize_normals / colorize_confidence (colorize.hpp:9-15,
 * colorize.cpp:32-70): rgb = 3*width*height bytes. */
int fmvs_colorize_depth(fmvs_ctx* ctx, const float* depth, int32_t width, int32_t height,
                        double lo, double hi, uint8_t* rgb);
int fmvs_colorize_normals(fmvs_ctx* ctx, const float* normals_xyz, int32_t width, int32_t height,
                          uint8_t* rgb);
int fmvs_colorize_confidence(fmvs_ctx* ctx, const float* confidence, int32_t width,
                             int32_t height, uint8_t* rgb);
/* write_pfm (map_io.hpp:25-26, map_io.cpp:34-44,95-113): channels 1 ("Pf",
 * depth / confidence) or 3 ("PF", normals xyz); rows written bottom to top,
 * little endian, byte-identical to the reference. InvalidInputError if the
 * file cannot be written. */
int fmvs_write_pfm(const char* path, const float* data, int32_t width, int32_t height,
                   int32_t channels);
/* write_png (map_io.hpp:27, map_io.cpp:203-260): 8-bit RGB, one IDAT chunk of
 * the filter-0 scanlines deflated by zlib at level 6 (compress2), CRC-32 per
 * chunk -- byte-identical to the reference with the same zlib.
 * rgb = 3*width*height bytes, row-major (the output of fmvs_colorize_*).
 * InvalidInputError if the file cannot be written or compression fails. */
int fmvs_write_png(const char* path, const uint8_t* rgb, int32_t width, int32_t height);

/* --------------------------------------- accuracy scoring -- */
/* L1Result + AccCplF (evaluation.hpp:11-30). */
typedef struct fmvs_l1_result {
    double l1_abs, l1_rel;
    uint64_t valid_both;
} fmvs_l1_result;
typedef struct fmvs_acc_cpl_f {
    double acc, cpl, f;
    uint64_t valid_both, valid_est, valid_gt;
} fmvs_acc_cpl_f;
/* evaluate (evaluation.hpp:48-49, evaluation.cpp:28-71,110-118): l1_metrics
 * + acc_cpl_f for n_thetas (<= 16) thresholds. Counts and ratios are exact;
 * the L1 means are FP64 tree sums (equal to the reference's sequential sum
 * up to FP64 rounding). InvalidInputError for empty / unequal maps or no
 * pixel valid in both. */
int fmvs_evaluate(fmvs_ctx* ctx, const float* est, const float* gt, int32_t width, int32_t height,
                  const double* thetas, int32_t n_thetas, fmvs_l1_result* l1,
                  fmvs_acc_cpl_f* scores);
/* roc_curve (evaluation.hpp:36-41, evaluation.cpp:73-108): densities and
 * error rates at 0.05, 0.10, ..., 1.00 (20 each), bit-identical. */
int fmvs_roc_curve(fmvs_ctx* ctx, const float* est, const float* gt, const float* confidence,
                   int32_t width, int32_t height, double theta, double* densities,
                   double* error_rates);

/* ------------------------------------- remaining reference helpers -- */
/* gaussian_blur (pipeline.hpp:54, pipeline.cpp:32-75): float raster, radius
 * <= 7. */
int fmvs_gaussian_blur(fmvs_ctx* ctx, const uint8_t* image, int32_t width, int32_t height,
                       int32_t radius, double sigma, float* out);
/* census_transform (matching.hpp:58, matching.cpp:44-55): u64 per pixel;
 * ConfigError for even windows or > 64 bits. */
int fmvs_census_transform(fmvs_ctx* ctx, const uint8_t* image, int32_t width, int32_t height,
                          int32_t window_w, int32_t window_h, uint64_t* out);
/* census_bits_at (matching.hpp:60, matching.cpp:28-42), host. */
uint64_t fmvs_census_bits_at(const uint8_t* image, int32_t width, int32_t height, int32_t x,
                             int32_t y, int32_t window_w, int32_t window_h);
/* ncc_cost (matching.hpp:64, matching.cpp:57-77), host: the standalone NCC
 * of two equal-size patches (the sweep uses its own two-pass form). */
int fmvs_ncc_cost(const float* patch_ref, const float* patch_other, int32_t n, int32_t* cost);
/* apply_homography (geometry.hpp:102, geometry.cpp:116-119), host. */
void fmvs_apply_homography(const double h[9], double x, double y, double out[2]);
/* cross_ratio (geometry.hpp:120-123, geometry.cpp:157-181), host: dims 2 or
 * 3, points packed p1..p4. InvalidInputError on coincident points. */
int fmvs_cross_ratio(const double* points, int32_t dims, double* out);
/* require_centers_in_front (geometry.hpp:115-116, geometry.cpp:147-153),
 * host: GeometryError when a camera centre lies behind the near plane. */
int fmvs_require_centers_in_front(const double normal[3], double delta_min,
                                  const double* centers_xyz, int32_t n);

#ifdef __cplusplus
}
#endif

#endif /* FMVS_H */
