// Host-callable launchers for the sm_100a kernels (one .cu per stage). All
// launchers enqueue on the given stream and never synchronise; the driver
// (driver.cpp) owns buffers and ordering.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

namespace fmvs {
namespace k {

// ---- K1: pyramid (pipeline.cpp:32-126) + quad packing for the sweep ------
// out(x,y) = clamp(lround(blur3x3(in)(2x,2y))) with reflected borders.
void blur_halve(const uint8_t* in, int win, int hin, uint8_t* out, int wout, int hout,
                const double k3[3], cudaStream_t s);
// quad[p] = I(x0,y0) | I(x1,y0)<<8 | I(x0,y1)<<16 | I(x1,y1)<<24, x1/y1 clamped:
// the four bilinear taps of raster.hpp:71-84 in one 32-bit load.
void pack_quads(const uint8_t* img, int w, int h, uint32_t* quad, cudaStream_t s);

// Batched launches (blockIdx.z = image): pyramid halving of up to kImgBatch
// images (in -> out) and quad packing (in -> quad, in sizes win x hin).
constexpr int kImgBatch = 32;
struct ImgJob {
    const uint8_t* in;
    uint8_t* out;
    uint32_t* quad;
    int win, hin, wout, hout;
};
struct ImgBatch {
    ImgJob job[kImgBatch];
};
void blur_halve_batch(const ImgBatch& b, int n, const double k3[3], cudaStream_t s);
void pack_quads_batch(const ImgBatch& b, int n, cudaStream_t s);

// ---- K3: per-pixel sampling range + plane interval + row prefix sums -----
struct RangeArgs {
    dev::Intr intr;
    double nx, ny, nz;           // sweep normal
    const double* planes;        // current level stack (device)
    int nplanes;
    int mode;                    // 0 uniform, 1 refine from prior, 2 explicit lo/hi
    double d_min, d_max;
    // mode 1 (refine_range, pipeline.cpp:136-173)
    const float* prior;          // coarser-level depth (device)
    int prior_w, prior_h;
    int policy;                  // FMVS_RANGE_*
    double policy_value;
    const double* coarser;       // coarser stack (device)
    int ncoarser;
    // mode 2
    const float* lo_in;
    const float* hi_in;
    // optional outputs of refine_range
    float* lo_out;
    float* hi_out;
    // outputs
    dev::VolMeta* meta;
    uint32_t* row_total;         // H entries
};
void range_rows(const RangeArgs& a, cudaStream_t s);
// row_base[y] = sum of row_total[0..y), row_base[H] = total entries.
void scan_rows(const uint32_t* row_total, int h, uint64_t* row_base, cudaStream_t s);
// agg[0 .. *count) = 0 (the SGM accumulator of a level; count on the device,
// 16-byte aligned agg).
void zero_entries(uint32_t* agg, const uint64_t* count, cudaStream_t s, bool agg16 = false);

// ---- K4: plane-sweep cost volume (matching.cpp:116-294) ------------------
struct SweepArgs {
    int w, h;                        // reference (level) size
    const uint8_t* ref_img;
    int nmatch;                      // matching views
    const uint32_t* const* quads;    // [nmatch] device pointers (device array)
    const int2* sizes;               // [nmatch] (w, h) (device array)
    const double* homs;              // [nmatch][nplanes][9] row-major (device)
    int nplanes;
    int nleft;                       // matching views left of the reference
    const dev::VolMeta* meta;
    const uint64_t* row_base;
    uint16_t* costs;
    int kind, ww, wh;
    const uint16_t* census_lut;      // [bits+1]
    // set by the launcher: pixels with count <= exact_above go to the tiled
    // certified census kernel, the rest to the exact per-hypothesis kernel
    int exact_above;
    int disable_tiled;               // force the exact per-hypothesis kernel
    int plane_slicing;               // dense ranges: split planes across CTAs (grid z); the
                                     // tiled kernels then stage each pixel's costs of 16
                                     // planes and write them as one 32-byte run
    int narrow_max;                  // pixels with more hypotheses take the exact kernel (0: default)
    int small_lists;                 // test hook (FMVS_NCC_SMALL_LISTS): NCC exact lists of 2 views / 2
                                     // pending entries, to exercise the overflow paths
    unsigned long long* stats;       // optional diagnostics (fmvs_ctx_sweep_stats)
};
// returns the number of kernels launched
int sweep(const SweepArgs& a, cudaStream_t s);


// ---- K5: surface-normal SGM shifts (sgm.cpp:252-299) ---------------------
struct OffsetArgs {
    dev::Intr intr;
    int w, h;
    const float* prior_depth;        // coarser level (upscaled on the fly) or same size
    const float* prior_normals;      // xyz
    int prior_w, prior_h;
    double nx, ny, nz;
    const double* planes;
    int nplanes;
    int16_t* out;                    // 4 per pixel
};
void normal_offsets(const OffsetArgs& a, cudaStream_t s);

// ---- K6: SGM path aggregation (sgm.cpp:91-239) ---------------------------
struct SgmArgs {
    int w, h;
    const dev::VolMeta* meta;
    const uint64_t* row_base;
    const uint16_t* costs;
    uint32_t* agg;
    const uint8_t* image;
    int variant;
    long long phi1;
    const long long* phi2_lut;       // [256] device
    long long phi2_max;              // max of the LUT (host), selects the int32 path
    const int16_t* offsets;          // SN shifts (4 per pixel) or null
    // PG (scene points)
    dev::Intr intr;
    double nx, ny, nz;
    const double* planes;
    int nplanes;
    int ndirs;
    int dirs[8][2];
    int pmax;                        // per-warp path buffer length
    uint32_t* scratch;               // global path buffers (2 x pmax per line)
    int group;                       // lanes per line for Plane/SN (4, 8, 32); 0 = 1 line/warp kernel
    int kper;                        // hypotheses per lane and pass (register blocking)
    int group_caps;                  // shared-memory path buffer length per line (grouped kernel)
    // Line kernel (unit directions, Plane/SN, int32 recurrence): scratch of
    // sgm_line_scratch_words(w, h) words for the per-pixel step records and
    // the wide-line flags, or null for the general kernel; an upper bound of
    // the level's entry count (the records hold 32-bit entry indices).
    uint32_t* line_scratch;
    uint64_t entries_bound;
    // packed aggregate: entry e is the u16 at index e of `agg` (two per 32-bit
    // word; set only when sgm_agg16_ok proved every sum fits 16 bits)
    int agg16;
    // upper bound of every matching cost in the volume (-1: unknown, u16)
    int cost_max;
};
// the line kernel runs this configuration (else the general kernel)
bool sgm_line_applicable(const SgmArgs& a);
bool sgm_fast32(const SgmArgs& a);
// a packed u16 aggregate is exact for this configuration, per-pixel matching
// costs <= cost_max
bool sgm_agg16_ok(const SgmArgs& a, long long cost_max);
void sgm(const SgmArgs& a, cudaStream_t s);
// entries every cost and aggregate allocation carries past the volume (the
// line kernel's inactive lanes add 0 there; its cost staging reads aligned
// 16-byte chunks that may extend up to 46 bytes past a pixel's last cost)
constexpr size_t kAggSlack = 256;  // >= the widest pass (G x K = 32 x 8)
size_t sgm_line_scratch_words(int w, int h);
// per-line global path buffers (SgmArgs::scratch): 2 x (pmax + kSgmLinePad)
// words per line (sentinel slots of either SGM kernel)
constexpr int kSgmLinePad = 32;
int sgm_total_lines(int w, int h, int ndirs);
// Lines of the given path directions (any step, sgm.cpp:213-219).
int sgm_lines(int w, int h, const int (*dirs)[2], int ndirs);

// ---- K7: WTA + depth + parabola (sgm.cpp:333-363, pipeline.cpp:263-288) ---
struct WtaArgs {
    int w, h;
    const dev::VolMeta* meta;
    const uint64_t* row_base;
    const uint32_t* agg;
    int agg16;                       // packed u16 aggregate (SgmArgs::agg16)
    int32_t* winners;                // optional
    float* depth;                    // optional (needs intr/planes)
    dev::Intr intr;
    double nx, ny, nz;
    const double* planes;
    int nplanes;
    int wide;                        // long ranges (dense levels): warp-cooperative scan
};
void wta_depth(const WtaArgs& a, cudaStream_t s);

// ---- K8/K9: per-pixel map kernels -----------------------------------------
void median5(const float* in, int w, int h, float* out, cudaStream_t s);
void normals_raw(const float* depth, int w, int h, dev::Intr intr, float* out_xyz,
                 cudaStream_t s);
// smooth_normals (+ confidence_map when conf != nullptr)
void smooth_conf(const float* raw_xyz, const uint8_t* img, int w, int h, int radius,
                 const double* weights, float* out_xyz, float* conf, double cos_rho,
                 double plane_dot_view, double nx, double ny, double nz, cudaStream_t s);
void confidence(const float* normals_xyz, int w, int h, double cos_rho, double plane_dot_view,
                double nx, double ny, double nz, float* out, cudaStream_t s);
void upscale(const float* in, int iw, int ih, int ch, float* out, int ow, int oh,
             cudaStream_t s);

// ---- post-filters (postfilter.cpp) -----------------------------------------
// gaussian_blur weights (pipeline.cpp:33-40), host-computed, radius <= 7
struct BlurKernel {
    int radius;
    double w[15];
};
// gaussian_blur(img) fused with the DoG activation |I - blur| > 0.5
// (postfilter.cpp:68-74); tmp: w*h floats
void gaussian_blur_dog(const uint8_t* img, int w, int h, const BlurKernel& k, float* tmp,
                       uint8_t* mask, cudaStream_t s);
// gaussian_blur (pipeline.cpp:32-75) -> float raster; tmp: w*h floats
void gaussian_blur(const uint8_t* img, int w, int h, const BlurKernel& k, float* tmp, float* out,
                   cudaStream_t s);
// census_transform (matching.cpp:44-55)
void census_transform(const uint8_t* img, int w, int h, int ww, int wh, uint64_t* out, cudaStream_t s);
// remove_speckles (postfilter.cpp:14-51): labels, sizes: w*h ints each
void remove_speckles(uint8_t* mask, int w, int h, uint8_t value, int min_size, int* labels,
                     int* sizes, cudaStream_t s);
void dilate3(const uint8_t* in, int w, int h, uint8_t* out, cudaStream_t s);
// apply_mask (postfilter.cpp:81-93) on device maps of n pixels
void apply_mask(float* depth, float* normals_xyz, float* conf, const uint8_t* mask, int n,
                cudaStream_t s);
struct GeomView {                    // ConsistencyView (postfilter.hpp:24-28)
    const float* depth;
    int w, h;
    dev::Intr k;
    double R[9];
    double C[3];
};
struct GeomArgs {
    const GeomView* views;           // device array
    int n, ref;
    double eta_r;
    int eta_h;
    int bilinear;                    // DepthLookup::Bilinear
    uint8_t* keep;
};
void geometric_mask(const GeomArgs& a, int w, int h, cudaStream_t s);

// ---- output stage (colorize.cpp) -------------------------------------------
// kind 0: viridis depth in [lo, hi]; 1: (n + 1) / 2 normals (xyz input);
// 2: gray confidence. rgb: 3 bytes per pixel.
void colorize(int kind, const float* in, int n, double lo, double hi, uint8_t* rgb, cudaStream_t s);

// ---- accuracy scoring (evaluation.cpp:28-124) -------------------------------
struct EvalThetas {
    int n;                           // <= 16
    double theta[16];
};
// counts: [valid_est, valid_gt, valid_both, pass(theta_0..n-1)];
// partials: 2 doubles per 256-pixel block; sums: {sum |e-g|, sum |e-g|/g}
void evaluate_counts(const float* est, const float* gt, int n, const EvalThetas& th,
                     unsigned long long* counts, double* partials, double* sums, cudaStream_t s);
struct RocSteps {
    long long m[20];                 // retained prefix length per density step
};
size_t roc_scratch_bytes(int n);
void roc_entries(const float* est, const float* gt, const float* conf, int n, double theta,
                 float* keys, uint8_t* pass, unsigned long long* count, cudaStream_t s);
void roc_sort_prefix(const float* keys, float* keys_sorted, const uint8_t* pass, uint8_t* pass_sorted,
                     int n, void* temp, size_t temp_bytes, const RocSteps& steps,
                     unsigned long long* prefix, cudaStream_t s);

// ---- synthetic input: render_scene (any planes, both textures) -------------
struct RenderPlane {
    double pt[3], n[3], u[3], v[3];  // PlaneFrame (normalised on the host)
    double ext_u, ext_v;
};
struct RenderArgs {
    int w, h;
    dev::Intr intr;
    double rot[9];                   // world -> camera rotation (row-major)
    double center[3];
    const RenderPlane* planes;       // device array
    int nplanes;
    int texture;                     // FMVS_TEXTURE_*
    double texture_scale;
    uint64_t seed;
    uint8_t* image;
    float* gt_depth;
    float* gt_normals;
};
void render_view(const RenderArgs& a, cudaStream_t s);

}  // namespace k
}  // namespace fmvs
