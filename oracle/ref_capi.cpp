// Oracle C ABI: the UNMODIFIED reference library (/root/reference/proj/src,
// built against oracle/eigen_shim by oracle/Makefile) exposed through the same
// signatures as include/fmvs.h with a `ref_` prefix, so the parity tests can
// drive the reference and the B200 library through one Python binding.
//
// TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
// CPU-baseline leg load this library. Nothing here is on the product path.
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <exception>
#include <limits>
#include <span>
#include <string>
#include <vector>

#include "fassmvs/errors.hpp"
#include "fassmvs/colorize.hpp"
#if __has_include(<json.hpp>)
#include "fassmvs/evaluation.hpp"
#define FMVS_REF_HAS_EVALUATION 1
#endif
#include "fassmvs/geometry.hpp"
#include "fassmvs/map_io.hpp"
#include "fassmvs/matching.hpp"
#include "fassmvs/parallel.hpp"
#include "fassmvs/pipeline.hpp"
#include "fassmvs/postfilter.hpp"
#include "fassmvs/render.hpp"
#include "fassmvs/sgm.hpp"
#include "fassmvs/surface.hpp"
#include "fmvs.h"

using namespace fassmvs;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return FMVS_OK;
    } catch (const InvalidInputError& e) {
        g_err = e.what();
        return FMVS_ERR_INVALID_INPUT;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return FMVS_ERR_CONFIG;
    } catch (const GeometryError& e) {
        g_err = e.what();
        return FMVS_ERR_GEOMETRY;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FMVS_ERR_CUDA;
    }
}

Intrinsics to_intr(const fmvs_intrinsics& i) {
    Intrinsics r;
    r.fx = i.fx;
    r.fy = i.fy;
    r.cx = i.cx;
    r.cy = i.cy;
    r.width = i.width;
    r.height = i.height;
    return r;
}

fmvs_intrinsics from_intr(const Intrinsics& i) {
    return {i.fx, i.fy, i.cx, i.cy, i.width, i.height};
}

Pose to_pose(const fmvs_pose& p) {
    Pose r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.rotation(i, j) = p.rotation[3 * i + j];
    r.center = Eigen::Vector3d(p.center[0], p.center[1], p.center[2]);
    return r;
}

fmvs_pose from_pose(const Pose& p) {
    fmvs_pose r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.rotation[3 * i + j] = p.rotation(i, j);
    for (int i = 0; i < 3; ++i)
        r.center[i] = p.center(i);
    return r;
}

ImageU8 to_image(const uint8_t* data, int w, int h) {
    ImageU8 img(w, h, 0);
    if (data && w > 0 && h > 0)
        std::memcpy(img.data(), data, static_cast<std::size_t>(w) * h);
    return img;
}

std::vector<CalibratedView> to_bundle(const fmvs_view* views, int n) {
    std::vector<CalibratedView> b(n);
    for (int k = 0; k < n; ++k) {
        b[k].intrinsics = to_intr(views[k].intrinsics);
        b[k].pose = to_pose(views[k].pose);
        b[k].image = to_image(views[k].image, views[k].intrinsics.width,
                              views[k].intrinsics.height);
    }
    return b;
}

Eigen::Vector3d v3(const double* n) { return Eigen::Vector3d(n[0], n[1], n[2]); }

PlaneStack to_stack(const fmvs_plane_stack* s) {
    PlaneStack p;
    p.normal = v3(s->normal);
    p.distances.assign(s->distances, s->distances + s->count);
    return p;
}

SgmConfig to_sgm(const fmvs_sgm_config& c) {
    SgmConfig s;
    s.variant = static_cast<SgmVariant>(c.variant);
    s.paths = c.paths;
    s.phi1 = c.phi1;
    s.phi2_adaptive = c.phi2_adaptive != 0;
    s.phi2_fixed = c.phi2_fixed;
    s.alpha = c.alpha;
    s.beta = c.beta;
    s.penalty_scale = c.penalty_scale;
    return s;
}

CostFunctionSpec to_cost(const fmvs_cost_spec& c) {
    CostFunctionSpec s;
    s.kind = static_cast<CostKind>(c.kind);
    s.window_w = c.window_w;
    s.window_h = c.window_h;
    return s;
}

PipelineConfig to_config(const fmvs_config& c) {
    PipelineConfig p(DepthBounds(c.d_min, c.d_max));
    p.bundle_size = c.bundle_size;
    p.pyramid_levels = c.pyramid_levels;
    p.sweep_normal = v3(c.sweep_normal);
    p.range_policy.kind = static_cast<RangePolicy::Kind>(c.range_kind);
    p.range_policy.value = c.range_value;
    p.max_planes = c.max_planes;
    p.sgm = to_sgm(c.sgm);
    p.cost = to_cost(c.cost);
    p.normal_smoothing_radius = c.normal_smoothing_radius;
    return p;
}

DepthMap to_depth(const float* d, int w, int h) {
    DepthMap m(w, h, 0.0f);
    std::memcpy(m.data(), d, sizeof(float) * static_cast<std::size_t>(w) * h);
    return m;
}

NormalMap to_normals(const float* xyz, int w, int h) {
    NormalMap m = make_normal_map(w, h);
    for (std::size_t p = 0; p < static_cast<std::size_t>(w) * h; ++p)
        m.data()[p] = Eigen::Vector3f(xyz[3 * p], xyz[3 * p + 1], xyz[3 * p + 2]);
    return m;
}

void write_normals(const NormalMap& m, float* xyz) {
    for (std::size_t p = 0; p < m.size(); ++p) {
        xyz[3 * p] = m.data()[p].x();
        xyz[3 * p + 1] = m.data()[p].y();
        xyz[3 * p + 2] = m.data()[p].z();
    }
}

CostVolume to_volume(int w, int h, const fmvs_plane_stack* planes, const int32_t* first,
                     const int32_t* count, const uint64_t* offset, const uint16_t* costs,
                     uint64_t total) {
    CostVolume v;
    v.width = w;
    v.height = h;
    v.planes = to_stack(planes);
    const std::size_t npx = static_cast<std::size_t>(w) * h;
    v.first.assign(first, first + npx);
    v.count.assign(count, count + npx);
    v.offset.assign(offset, offset + npx);
    v.costs.assign(costs, costs + total);
    return v;
}

// ---- stage capture (tests/test_fullsize_gpu.py) ---------------------------
// A staged restatement of estimate_bundle (pipeline.cpp:200-309) through the
// reference's public stage functions, keeping one level's ragged layout,
// costs, aggregate, winners and pre-median depth. Its final maps are checked
// against the reference's own estimate_bundle before anything is reported.
struct Capture {
    int level = -1;
    int w = 0, h = 0;
    std::vector<int32_t> first, count, winners;
    std::vector<uint64_t> offset;
    std::vector<uint16_t> costs;
    std::vector<uint32_t> agg;
    std::vector<float> depth_raw;
};
thread_local Capture g_cap;

BundleResult estimate_bundle_staged(const std::vector<CalibratedView>& bundle,
                                    const PipelineConfig& config, Capture* cap) {
    config.validate();
    if (bundle.size() < 3 || bundle.size() % 2 == 0)
        throw InvalidInputError("estimate: bundle must hold an odd number (>= 3) of views");
    const int ref_index = static_cast<int>(bundle.size()) / 2;
    const int n = config.pyramid_levels;
    const PyramidLevelSet pyr = build_pyramids(bundle, n);
    DepthMap prior_depth;
    NormalMap prior_normals;
    PlaneStack coarser;
    BundleResult out;
    for (int l = n - 1; l >= 0; --l) {
        const auto& views = pyr.levels[l];
        const Intrinsics& intr = views[ref_index].intrinsics;
        const int w = intr.width, h = intr.height;
        const auto [dlo, dhi] = bounding_distances(config.depth_bounds, config.sweep_normal, intr);
        int far = ref_index == 0 ? 1 : 0;
        double best = -1.0;
        for (int k = 0; k < static_cast<int>(views.size()); ++k) {
            const double d = k == ref_index ? -1.0 : (views[k].pose.center - views[ref_index].pose.center).norm();
            if (k != ref_index && d > best) {
                best = d;
                far = k;
            }
        }
        PlaneStack stack;
        stack.normal = config.sweep_normal;
        stack.distances = plane_distances(intr, views[ref_index].pose, views[far].intrinsics,
                                          views[far].pose, dlo, dhi, config.sweep_normal,
                                          l == n - 1 ? config.max_planes : std::numeric_limits<int>::max());
        const bool prior = l < n - 1;
        const SamplingRange ranges =
            prior ? refine_range(prior_depth, config.range_policy, config.depth_bounds, &coarser, &intr)
                  : SamplingRange::uniform(config.depth_bounds, w, h);
        const CostVolume vol = sweep_cost_volume(views, ref_index, stack, ranges, config.cost);
        SgmConfig sc = config.sgm;
        sc.penalty_scale = static_cast<int>(bundle.size()) / 2;
        if (sc.variant == SgmVariant::SurfaceNormal && !prior)
            sc.variant = SgmVariant::Plane;
        const AggregatedVolume agg = aggregate(vol, views[ref_index].image, sc, intr,
                                               prior ? &prior_normals : nullptr,
                                               prior ? &prior_depth : nullptr);
        const PlaneIndexMap win = wta(agg);
        DepthMap depth(w, h, 0.0f);
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                const int32_t i = win.at(x, y);
                if (i < 0)
                    continue;
                const Eigen::Vector2d px(x, y);
                const double dw = depth_from_plane(px, stack.plane(i), intr);
                if (dw <= 0.0)
                    continue;
                const std::size_t p = agg.pixel(x, y);
                const int32_t f = agg.first[p];
                double d = dw;
                if (i - 1 >= f && i + 1 < f + agg.count[p]) {
                    const uint32_t* v = agg.values.data() + agg.offset[p];
                    const double a = depth_from_plane(px, stack.plane(i + 1), intr);
                    const double c = depth_from_plane(px, stack.plane(i - 1), intr);
                    if (a > 0.0 && c > 0.0 && a < dw && dw < c)
                        d = parabola_refine(a, dw, c, v[i + 1 - f], v[i - f], v[i - 1 - f]);
                }
                depth.at(x, y) = static_cast<float>(d);
            }
        if (cap && cap->level == l) {
            cap->w = w;
            cap->h = h;
            cap->first.assign(vol.first.begin(), vol.first.end());
            cap->count.assign(vol.count.begin(), vol.count.end());
            cap->offset.assign(vol.offset.begin(), vol.offset.end());
            cap->costs.assign(vol.costs.begin(), vol.costs.end());
            cap->agg.assign(agg.values.begin(), agg.values.end());
            cap->winners.assign(win.data(), win.data() + win.size());
            cap->depth_raw.assign(depth.data(), depth.data() + depth.size());
        }
        depth = median_filter_5x5(depth);
        NormalMap normals = smooth_normals(normals_from_depth(depth, intr), views[ref_index].image,
                                           config.normal_smoothing_radius);
        ConfidenceMap conf = confidence_map(normals, config.sweep_normal);
        if (l > 0) {
            const Intrinsics& next = pyr.levels[l - 1][ref_index].intrinsics;
            prior_depth = upscale_nearest(depth, next.width, next.height);
            prior_normals = upscale_nearest(normals, next.width, next.height);
            coarser = stack;
        } else {
            out.depth = std::move(depth);
            out.normals = std::move(normals);
            out.confidence = std::move(conf);
        }
    }
    return out;
}

}  // namespace

extern "C" {

int32_t ref_abi_version(void) { return FMVS_ABI_VERSION; }

// Same contract as fmvs_ctx_set_capture / fmvs_ctx_capture_* (include/fmvs.h).
int ref_ctx_set_capture(void*, int32_t level) {
    g_cap = Capture{};
    g_cap.level = level;
    return FMVS_OK;
}

int ref_ctx_capture_sizes(void*, int32_t* w, int32_t* h, uint64_t* entries) {
    if (g_cap.w == 0) {
        g_err = "capture: nothing captured";
        return FMVS_ERR_INVALID_INPUT;
    }
    *w = g_cap.w;
    *h = g_cap.h;
    *entries = g_cap.costs.size();
    return FMVS_OK;
}

int ref_ctx_capture_copy(void*, int32_t* first, int32_t* count, uint64_t* offset, uint16_t* costs,
                         uint32_t* agg, int32_t* winners, float* depth_raw) {
    if (g_cap.w == 0) {
        g_err = "capture: nothing captured";
        return FMVS_ERR_INVALID_INPUT;
    }
    std::copy(g_cap.first.begin(), g_cap.first.end(), first);
    std::copy(g_cap.count.begin(), g_cap.count.end(), count);
    std::copy(g_cap.offset.begin(), g_cap.offset.end(), offset);
    std::copy(g_cap.costs.begin(), g_cap.costs.end(), costs);
    std::copy(g_cap.agg.begin(), g_cap.agg.end(), agg);
    std::copy(g_cap.winners.begin(), g_cap.winners.end(), winners);
    std::copy(g_cap.depth_raw.begin(), g_cap.depth_raw.end(), depth_raw);
    return FMVS_OK;
}
const char* ref_last_error(void) { return g_err.c_str(); }

int ref_worker_count(void) { return worker_count(); }

void ref_config_default(fmvs_config* cfg, double d_min, double d_max) {
    const PipelineConfig p(DepthBounds(d_min, d_max));
    cfg->bundle_size = p.bundle_size;
    cfg->pyramid_levels = p.pyramid_levels;
    cfg->d_min = d_min;
    cfg->d_max = d_max;
    for (int i = 0; i < 3; ++i)
        cfg->sweep_normal[i] = p.sweep_normal(i);
    cfg->range_kind = static_cast<int32_t>(p.range_policy.kind);
    cfg->range_value = p.range_policy.value;
    cfg->max_planes = p.max_planes;
    cfg->sgm = {static_cast<int32_t>(p.sgm.variant), p.sgm.paths, p.sgm.phi1,
                p.sgm.phi2_adaptive ? 1 : 0, p.sgm.phi2_fixed, p.sgm.alpha, p.sgm.beta,
                p.sgm.penalty_scale};
    cfg->cost = {static_cast<int32_t>(p.cost.kind), p.cost.window_w, p.cost.window_h};
    cfg->normal_smoothing_radius = p.normal_smoothing_radius;
}

int ref_estimate_bundle(void*, const fmvs_view* views, int32_t n_views, const fmvs_config* cfg,
                        float* depth, float* normals_xyz, float* confidence) {
    return guard([&] {
        const std::vector<CalibratedView> bundle = to_bundle(views, n_views);
        const PipelineConfig config = to_config(*cfg);
        const BundleResult r = estimate_bundle(bundle, config);
        if (g_cap.level >= 0) {
            const BundleResult s = estimate_bundle_staged(bundle, config, &g_cap);
            auto same = [](const auto& a, const auto& b, std::size_t bytes) {
                return std::memcmp(a.data(), b.data(), bytes) == 0;
            };
            const std::size_t px = r.depth.size();
            if (s.depth.size() != px || !same(s.depth, r.depth, 4 * px) ||
                !same(s.confidence, r.confidence, 4 * px) ||
                !same(s.normals, r.normals, sizeof(Eigen::Vector3f) * px))
                throw std::runtime_error("capture: staged restatement differs from estimate_bundle");
            g_cap.level = -1;
        }
        std::memcpy(depth, r.depth.data(), sizeof(float) * r.depth.size());
        write_normals(r.normals, normals_xyz);
        std::memcpy(confidence, r.confidence.data(), sizeof(float) * r.confidence.size());
    });
}

int ref_plane_homography(const double normal[3], double distance, const fmvs_intrinsics* ri,
                         const fmvs_pose* rp, const fmvs_intrinsics* oi, const fmvs_pose* op,
                         double out_h[9]) {
    return guard([&] {
        const Eigen::Matrix3d h = plane_homography(SweepPlane{v3(normal), distance}, to_intr(*ri),
                                                   to_pose(*rp), to_intr(*oi), to_pose(*op));
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                out_h[3 * i + j] = h(i, j);
    });
}

int ref_bounding_distances(double d_min, double d_max, const double normal[3],
                           const fmvs_intrinsics* ri, double* dmin, double* dmax) {
    return guard([&] {
        const auto [a, b] = bounding_distances(DepthBounds(d_min, d_max), v3(normal), to_intr(*ri));
        *dmin = a;
        *dmax = b;
    });
}

int ref_plane_distances(const fmvs_intrinsics* ri, const fmvs_pose* rp, const fmvs_intrinsics* oi,
                        const fmvs_pose* op, double delta_min, double delta_max,
                        const double normal[3], int32_t max_planes, double* out,
                        int32_t capacity, int32_t* count) {
    int rc = guard([&] {
        const std::vector<double> d = plane_distances(to_intr(*ri), to_pose(*rp), to_intr(*oi),
                                                      to_pose(*op), delta_min, delta_max,
                                                      v3(normal), max_planes);
        *count = static_cast<int32_t>(d.size());
        for (int i = 0; i < static_cast<int>(d.size()) && i < capacity; ++i)
            out[i] = d[i];
    });
    if (rc == FMVS_OK && *count > capacity) {
        g_err = "plane distances: output capacity too small";
        return FMVS_ERR_CAPACITY;
    }
    return rc;
}

double ref_depth_from_plane(double x, double y, const double normal[3], double distance,
                            const fmvs_intrinsics* intr) {
    return depth_from_plane(Eigen::Vector2d(x, y), SweepPlane{v3(normal), distance},
                            to_intr(*intr));
}

double ref_adaptive_phi2(double phi1, double alpha, double beta, double di) {
    return adaptive_phi2(phi1, alpha, beta, di);
}

int ref_parabola_refine(double a, double b, double c, double ca, double cb, double cc,
                        double* out) {
    return guard([&] { *out = parabola_refine(a, b, c, ca, cb, cc); });
}

int ref_build_pyramids(void*, const fmvs_view* views, int32_t n_views, int32_t levels,
                       uint8_t* out_images, uint64_t capacity, fmvs_intrinsics* out_intr) {
    return guard([&] {
        const PyramidLevelSet set = build_pyramids(to_bundle(views, n_views), levels);
        uint64_t pos = 0;
        for (int l = 0; l < levels; ++l)
            for (int k = 0; k < n_views; ++k) {
                const CalibratedView& v = set.levels[l][k];
                out_intr[l * n_views + k] = from_intr(v.intrinsics);
                if (pos + v.image.size() > capacity)
                    throw std::runtime_error("pyramid output capacity too small");
                std::memcpy(out_images + pos, v.image.data(), v.image.size());
                pos += v.image.size();
            }
    });
}

int ref_gaussian_blur(void*, const uint8_t* image, int32_t w, int32_t h, int32_t radius, double sigma,
                      float* out) {
    return guard([&] {
        const Raster<float> r = gaussian_blur(to_image(image, w, h), radius, sigma);
        std::memcpy(out, r.data(), sizeof(float) * r.size());
    });
}

int ref_refine_range(void*, const float* prior, int32_t w, int32_t h, int32_t kind, double value,
                     double d_min, double d_max, const fmvs_plane_stack* coarser,
                     const fmvs_intrinsics* intr, float* lo, float* hi) {
    return guard([&] {
        RangePolicy pol;
        pol.kind = static_cast<RangePolicy::Kind>(kind);
        pol.value = value;
        PlaneStack stack;
        if (coarser)
            stack = to_stack(coarser);
        Intrinsics in;
        if (intr)
            in = to_intr(*intr);
        const SamplingRange r = refine_range(to_depth(prior, w, h), pol, DepthBounds(d_min, d_max),
                                             coarser ? &stack : nullptr, intr ? &in : nullptr);
        std::memcpy(lo, r.lo.data(), sizeof(float) * r.lo.size());
        std::memcpy(hi, r.hi.data(), sizeof(float) * r.hi.size());
    });
}

int ref_sweep_cost_volume(void*, const fmvs_view* views, int32_t n_views, int32_t ref_index,
                          const fmvs_plane_stack* planes, const float* lo, const float* hi,
                          const fmvs_cost_spec* cost, int32_t* first, int32_t* count,
                          uint64_t* offset, uint16_t* costs, uint64_t capacity, uint64_t* total,
                          int32_t* per_side) {
    int rc = guard([&] {
        const std::vector<CalibratedView> b = to_bundle(views, n_views);
        const int w = b[ref_index < 0 || ref_index >= n_views ? 0 : ref_index].intrinsics.width;
        const int h = b[ref_index < 0 || ref_index >= n_views ? 0 : ref_index].intrinsics.height;
        SamplingRange r;
        r.lo = to_depth(lo, w, h);
        r.hi = to_depth(hi, w, h);
        const CostVolume v = sweep_cost_volume(b, ref_index, to_stack(planes), r, to_cost(*cost));
        const std::size_t npx = static_cast<std::size_t>(w) * h;
        std::memcpy(first, v.first.data(), 4 * npx);
        std::memcpy(count, v.count.data(), 4 * npx);
        for (std::size_t p = 0; p < npx; ++p)
            offset[p] = v.offset[p];
        *total = v.costs.size();
        *per_side = v.per_side;
        if (v.costs.size() <= capacity)
            std::memcpy(costs, v.costs.data(), 2 * v.costs.size());
    });
    if (rc == FMVS_OK && *total > capacity) {
        g_err = "sweep: cost capacity too small";
        return FMVS_ERR_CAPACITY;
    }
    return rc;
}

int ref_compute_normal_offsets(void*, const float* prior_normals_xyz, const float* prior_depth,
                               int32_t w, int32_t h, const fmvs_plane_stack* planes,
                               const fmvs_intrinsics* intr, int16_t* out) {
    return guard([&] {
        const NormalOffsets o = compute_normal_offsets(to_normals(prior_normals_xyz, w, h),
                                                       to_depth(prior_depth, w, h),
                                                       to_stack(planes), to_intr(*intr));
        for (std::size_t p = 0; p < o.size(); ++p)
            for (int c = 0; c < 4; ++c)
                out[4 * p + c] = o.data()[p][c];
    });
}

int ref_aggregate(void*, int32_t w, int32_t h, const fmvs_plane_stack* planes,
                  const int32_t* first, const int32_t* count, const uint64_t* offset,
                  const uint16_t* costs, uint64_t total, const uint8_t* image,
                  const fmvs_sgm_config* cfg, const fmvs_intrinsics* intr,
                  const float* prior_normals_xyz, const float* prior_depth, int32_t dir_x,
                  int32_t dir_y, uint32_t* out_values) {
    return guard([&] {
        const CostVolume v = to_volume(w, h, planes, first, count, offset, costs, total);
        NormalMap pn;
        DepthMap pd;
        if (prior_normals_xyz)
            pn = to_normals(prior_normals_xyz, w, h);
        if (prior_depth)
            pd = to_depth(prior_depth, w, h);
        const ImageU8 img = to_image(image, w, h);
        const Intrinsics in = to_intr(*intr);
        const AggregatedVolume a =
            (dir_x == 0 && dir_y == 0)
                ? aggregate(v, img, to_sgm(*cfg), in, prior_normals_xyz ? &pn : nullptr,
                            prior_depth ? &pd : nullptr)
                : aggregate_single_path(v, img, to_sgm(*cfg), in, dir_x, dir_y,
                                        prior_normals_xyz ? &pn : nullptr,
                                        prior_depth ? &pd : nullptr);
        std::memcpy(out_values, a.values.data(), 4 * a.values.size());
    });
}

int ref_aggregate_single_path(void*, int32_t w, int32_t h, const fmvs_plane_stack* planes,
                              const int32_t* first, const int32_t* count, const uint64_t* offset,
                              const uint16_t* costs, uint64_t total, const uint8_t* image,
                              const fmvs_sgm_config* cfg, const fmvs_intrinsics* intr,
                              const float* prior_normals_xyz, const float* prior_depth, int32_t dir_x,
                              int32_t dir_y, uint32_t* out_values) {
    return guard([&] {
        const CostVolume v = to_volume(w, h, planes, first, count, offset, costs, total);
        NormalMap pn;
        DepthMap pd;
        if (prior_normals_xyz)
            pn = to_normals(prior_normals_xyz, w, h);
        if (prior_depth)
            pd = to_depth(prior_depth, w, h);
        const AggregatedVolume a =
            aggregate_single_path(v, to_image(image, w, h), to_sgm(*cfg), to_intr(*intr), dir_x, dir_y,
                                  prior_normals_xyz ? &pn : nullptr, prior_depth ? &pd : nullptr);
        std::memcpy(out_values, a.values.data(), 4 * a.values.size());
    });
}

int ref_wta(void*, int32_t w, int32_t h, const int32_t* first, const int32_t* count,
            const uint64_t* offset, const uint32_t* values, uint64_t total, int32_t* winners) {
    return guard([&] {
        AggregatedVolume a;
        a.width = w;
        a.height = h;
        const std::size_t npx = static_cast<std::size_t>(w) * h;
        a.first.assign(first, first + npx);
        a.count.assign(count, count + npx);
        a.offset.assign(offset, offset + npx);
        a.values.assign(values, values + total);
        const PlaneIndexMap m = wta(a);
        std::memcpy(winners, m.data(), 4 * npx);
    });
}

int ref_median_filter_5x5(void*, const float* depth, int32_t w, int32_t h, float* out) {
    return guard([&] {
        const DepthMap m = median_filter_5x5(to_depth(depth, w, h));
        std::memcpy(out, m.data(), sizeof(float) * m.size());
    });
}

int ref_normals_from_depth(void*, const float* depth, int32_t w, int32_t h,
                           const fmvs_intrinsics* intr, float* out_xyz) {
    return guard([&] { write_normals(normals_from_depth(to_depth(depth, w, h), to_intr(*intr)), out_xyz); });
}

int ref_smooth_normals(void*, const float* raw_xyz, const uint8_t* image, int32_t w, int32_t h,
                       int32_t radius, float* out_xyz) {
    return guard([&] {
        write_normals(smooth_normals(to_normals(raw_xyz, w, h), to_image(image, w, h), radius),
                      out_xyz);
    });
}

int ref_confidence_map(void*, const float* normals_xyz, int32_t w, int32_t h,
                       const double sweep_normal[3], double rho_degrees, float* out) {
    return guard([&] {
        const ConfidenceMap c = confidence_map(to_normals(normals_xyz, w, h), v3(sweep_normal),
                                               rho_degrees);
        std::memcpy(out, c.data(), sizeof(float) * c.size());
    });
}

int ref_upscale_nearest(void*, const float* in, int32_t iw, int32_t ih, int32_t channels,
                        int32_t ow, int32_t oh, float* out) {
    return guard([&] {
        if (channels == 1) {
            const DepthMap m = upscale_nearest(to_depth(in, iw, ih), ow, oh);
            std::memcpy(out, m.data(), sizeof(float) * m.size());
        } else {
            write_normals(upscale_nearest(to_normals(in, iw, ih), ow, oh), out);
        }
    });
}

int ref_render_plane_scene(void*, int32_t kind, int32_t w, int32_t h, double focal, double depth,
                           double tilt_deg, int32_t n_views, double step, uint64_t seed,
                           double texture_scale, uint8_t* images, float* gt_depth,
                           float* gt_normals_xyz, fmvs_intrinsics* intr, fmvs_pose* poses) {
    return guard([&] {
        SyntheticScene s = kind == 0
                               ? fronto_scene(w, h, focal, depth, n_views, step, seed)
                               : slanted_scene(w, h, focal, depth, tilt_deg, n_views, step, seed);
        s.texture_scale = texture_scale;
        const std::vector<RenderedView> r = render_scene(s);
        const std::size_t npx = static_cast<std::size_t>(w) * h;
        for (int k = 0; k < n_views; ++k) {
            std::memcpy(images + k * npx, r[k].view.image.data(), npx);
            if (gt_depth)
                std::memcpy(gt_depth + k * npx, r[k].gt_depth.data(), 4 * npx);
            if (gt_normals_xyz)
                write_normals(r[k].gt_normals, gt_normals_xyz + 3 * k * npx);
            if (intr)
                intr[k] = from_intr(r[k].view.intrinsics);
            if (poses)
                poses[k] = from_pose(r[k].view.pose);
        }
    });
}

// render_scene (render.hpp:41-48) for an arbitrary SyntheticScene.
int ref_render_scene(void*, const fmvs_scene_plane* planes, int32_t n_planes, const fmvs_pose* poses,
                     int32_t n_poses, const fmvs_intrinsics* intr, int32_t texture, double texture_scale,
                     uint64_t seed, uint8_t* images, float* gt_depth, float* gt_normals_xyz) {
    return guard([&] {
        SyntheticScene s;
        for (int i = 0; i < n_planes; ++i) {
            ScenePlane sp;
            sp.point = Eigen::Vector3d(planes[i].point[0], planes[i].point[1], planes[i].point[2]);
            sp.normal = Eigen::Vector3d(planes[i].normal[0], planes[i].normal[1], planes[i].normal[2]);
            sp.u_axis = Eigen::Vector3d(planes[i].u_axis[0], planes[i].u_axis[1], planes[i].u_axis[2]);
            sp.extent_u = planes[i].extent_u;
            sp.extent_v = planes[i].extent_v;
            s.planes.push_back(sp);
        }
        for (int i = 0; i < n_poses; ++i)
            s.poses.push_back(to_pose(poses[i]));
        s.intrinsics = to_intr(*intr);
        s.texture = texture == FMVS_TEXTURE_CHECKERBOARD ? TextureKind::Checkerboard : TextureKind::ValueNoise;
        s.texture_scale = texture_scale;
        s.seed = seed;
        const std::vector<RenderedView> r = render_scene(s);
        const std::size_t npx = static_cast<std::size_t>(intr->width) * intr->height;
        for (int k = 0; k < n_poses; ++k) {
            std::memcpy(images + k * npx, r[k].view.image.data(), npx);
            if (gt_depth)
                std::memcpy(gt_depth + k * npx, r[k].gt_depth.data(), 4 * npx);
            if (gt_normals_xyz)
                write_normals(r[k].gt_normals, gt_normals_xyz + 3 * k * npx);
        }
    });
}

// --- post-filters (postfilter.hpp) and the CLI estimate loop ------------


// dog_mask (postfilter.hpp:18, postfilter.cpp:67-79).
int ref_dog_mask(void*, const uint8_t* image, int32_t w, int32_t h, uint8_t* out) {
    return guard([&] {
        const TextureMask m = dog_mask(to_image(image, w, h));
        for (std::size_t p = 0; p < m.size(); ++p)
            out[p] = m.data()[p] ? 1 : 0;
    });
}

// apply_mask (postfilter.hpp:21-22), in place.
int ref_apply_mask(void*, float* depth, float* normals_xyz, float* confidence, int32_t w, int32_t h,
                   const uint8_t* mask) {
    return guard([&] {
        DepthMap d = to_depth(depth, w, h);
        NormalMap n = make_normal_map(w, h);
        for (int i = 0; i < w * h; ++i)
            n.data()[i] = Eigen::Vector3f(normals_xyz[3 * i], normals_xyz[3 * i + 1], normals_xyz[3 * i + 2]);
        ConfidenceMap c = to_depth(confidence, w, h);
        TextureMask m(w, h, 0);
        std::memcpy(m.data(), mask, static_cast<std::size_t>(w) * h);
        apply_mask(d, n, c, m);
        std::memcpy(depth, d.data(), sizeof(float) * d.size());
        write_normals(n, normals_xyz);
        std::memcpy(confidence, c.data(), sizeof(float) * c.size());
    });
}

void ref_geom_filter_config_default(fmvs_geom_filter_config* c) {
    const GeomFilterConfig g;
    c->eta_r = g.eta_r;
    c->eta_h = g.eta_h;
    c->lookup = g.lookup == DepthLookup::Bilinear ? FMVS_LOOKUP_BILINEAR : FMVS_LOOKUP_NEAREST;
}

// geometric_consistency_mask (postfilter.hpp:44-45, postfilter.cpp:95-160).
int ref_geometric_consistency_mask(void*, const fmvs_consistency_view* window, int32_t n,
                                   int32_t ref_index, const fmvs_geom_filter_config* cfg,
                                   uint8_t* keep) {
    return guard([&] {
        std::vector<ConsistencyView> win(n);
        for (int i = 0; i < n; ++i)
            win[i] = {to_depth(window[i].depth, window[i].width, window[i].height),
                      to_intr(window[i].intrinsics), to_pose(window[i].pose)};
        GeomFilterConfig g;
        if (cfg) {
            g.eta_r = cfg->eta_r;
            g.eta_h = cfg->eta_h;
            g.lookup = cfg->lookup == FMVS_LOOKUP_BILINEAR ? DepthLookup::Bilinear : DepthLookup::Nearest;
        }
        const TextureMask m = geometric_consistency_mask(win, ref_index, g);
        for (std::size_t p = 0; p < m.size(); ++p)
            keep[p] = m.data()[p] ? 1 : 0;
    });
}

// The `fassmvs estimate` loop (tools/fassmvs.cpp:92-176) restated with the
// reference's own library calls, minus file I/O and the report: the oracle of
// fmvs_estimate_sequence.
int ref_estimate_sequence(void*, const fmvs_view* frames_c, int32_t n_frames, int32_t stride,
                          const fmvs_config* cfg, int32_t filter, float* depth, float* normals_xyz,
                          float* confidence, int32_t* ref_frames, int32_t capacity,
                          int32_t* n_results) {
    if (n_results)
        *n_results = 0;
    return guard([&] {
        if (cfg->bundle_size < 3 || cfg->bundle_size % 2 == 0)
            throw ConfigError("--bundle-size must be odd and at least 3");
        if (stride < 1)
            throw ConfigError("--stride must be at least 1");
        if (filter < 0 || filter > 3)
            throw ConfigError("--filter must be none, dog, geom or both");
        const PipelineConfig config = to_config(*cfg);
        config.validate();
        std::vector<CalibratedView> frames = to_bundle(frames_c, n_frames);
        for (auto& v : frames)
            v.validate();
        if (static_cast<int>(frames.size()) < config.bundle_size)
            throw InvalidInputError("sequence shorter than one bundle");
        const int half = config.bundle_size / 2;
        struct FrameResult {
            int frame;
            BundleResult maps;
        };
        std::vector<FrameResult> results;
        for (int ref = half; ref + half < static_cast<int>(frames.size()); ref += stride) {
            std::vector<CalibratedView> bundle(frames.begin() + (ref - half),
                                               frames.begin() + (ref + half + 1));
            results.push_back({ref, estimate_bundle(bundle, config)});
        }
        const int m = static_cast<int>(results.size());
        if (n_results)
            *n_results = m;
        if (m > capacity)
            throw std::runtime_error("capacity");
        if (filter == 1 || filter == 3)
            for (auto& r : results) {
                const TextureMask mask = dog_mask(frames[r.frame].image);
                apply_mask(r.maps.depth, r.maps.normals, r.maps.confidence, mask);
            }
        if (filter == 2 || filter == 3) {
            const int window_size = std::min(5, m);
            std::vector<TextureMask> masks(m);
            for (int i = 0; i < m; ++i) {
                const int start = std::clamp(i - window_size / 2, 0, m - window_size);
                std::vector<ConsistencyView> window;
                for (int k = start; k < start + window_size; ++k)
                    window.push_back({results[k].maps.depth, frames[results[k].frame].intrinsics,
                                      frames[results[k].frame].pose});
                masks[i] = geometric_consistency_mask(window, i - start);
            }
            for (int i = 0; i < m; ++i)
                apply_mask(results[i].maps.depth, results[i].maps.normals, results[i].maps.confidence,
                           masks[i]);
        }
        std::size_t px = 0;
        for (int r = 0; r < m; ++r) {
            const BundleResult& b = results[r].maps;
            px = b.depth.size();
            std::memcpy(depth + r * px, b.depth.data(), sizeof(float) * px);
            write_normals(b.normals, normals_xyz + 3 * r * px);
            std::memcpy(confidence + r * px, b.confidence.data(), sizeof(float) * px);
            ref_frames[r] = results[r].frame;
        }
    });
}

// --- output stage: colorize.hpp / map_io.hpp ---------------------------

void write_rgb(const RgbImage& img, uint8_t* rgb) {
    for (std::size_t p = 0; p < img.size(); ++p)
        for (int c = 0; c < 3; ++c)
            rgb[3 * p + c] = img.data()[p][c];
}

int ref_colorize_depth(void*, const float* depth, int32_t w, int32_t h, double lo, double hi,
                       uint8_t* rgb) {
    return guard([&] { write_rgb(colorize_depth(to_depth(depth, w, h), lo, hi), rgb); });
}

int ref_colorize_normals(void*, const float* normals_xyz, int32_t w, int32_t h, uint8_t* rgb) {
    return guard([&] { write_rgb(colorize_normals(to_normals(normals_xyz, w, h)), rgb); });
}

int ref_colorize_confidence(void*, const float* conf, int32_t w, int32_t h, uint8_t* rgb) {
    return guard([&] { write_rgb(colorize_confidence(to_depth(conf, w, h)), rgb); });
}

#ifdef FMVS_REF_HAS_EVALUATION
// --- accuracy scoring (evaluation.hpp) -------------------------------------
int ref_evaluate(void*, const float* est, const float* gt, int32_t w, int32_t h,
                 const double* thetas, int32_t n_thetas, fmvs_l1_result* l1, fmvs_acc_cpl_f* scores) {
    return guard([&] {
        const MetricReport r = evaluate(to_depth(est, w, h), to_depth(gt, w, h),
                                        std::vector<double>(thetas, thetas + n_thetas));
        l1->l1_abs = r.l1.l1_abs;
        l1->l1_rel = r.l1.l1_rel;
        l1->valid_both = r.l1.valid_both;
        for (int i = 0; i < n_thetas; ++i)
            scores[i] = {r.scores[i].acc, r.scores[i].cpl, r.scores[i].f, r.scores[i].valid_both,
                         r.scores[i].valid_est, r.scores[i].valid_gt};
    });
}

int ref_roc_curve(void*, const float* est, const float* gt, const float* conf, int32_t w, int32_t h,
                  double theta, double* densities, double* error_rates) {
    return guard([&] {
        const RocCurve c = roc_curve(to_depth(est, w, h), to_depth(gt, w, h), to_depth(conf, w, h), theta);
        for (std::size_t i = 0; i < c.densities.size(); ++i) {
            densities[i] = c.densities[i];
            error_rates[i] = c.error_rates[i];
        }
    });
}
#endif

// --- remaining reference helpers (matching.hpp / geometry.hpp) -----------

int ref_census_transform(void*, const uint8_t* image, int32_t w, int32_t h, int32_t ww, int32_t wh,
                         uint64_t* out) {
    return guard([&] {
        const Raster<std::uint64_t> r = census_transform(to_image(image, w, h), ww, wh);
        std::memcpy(out, r.data(), sizeof(uint64_t) * r.size());
    });
}

uint64_t ref_census_bits_at(const uint8_t* image, int32_t w, int32_t h, int32_t x, int32_t y, int32_t ww,
                            int32_t wh) {
    return census_bits_at(to_image(image, w, h), x, y, ww, wh);
}

int ref_ncc_cost(const float* a, const float* b, int32_t n, int32_t* cost) {
    return guard([&] {
        *cost = ncc_cost(std::span<const float>(a, static_cast<std::size_t>(std::max(n, 0))),
                         std::span<const float>(b, static_cast<std::size_t>(std::max(n, 0))));
    });
}

void ref_apply_homography(const double h[9], double x, double y, double out[2]) {
    Eigen::Matrix3d m;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            m(r, c) = h[3 * r + c];
    const Eigen::Vector2d q = apply_homography(m, Eigen::Vector2d(x, y));
    out[0] = q.x();
    out[1] = q.y();
}

int ref_cross_ratio(const double* p, int32_t dims, double* out) {
    return guard([&] {
        if (dims == 2)
            *out = cross_ratio(Eigen::Vector2d(p[0], p[1]), Eigen::Vector2d(p[2], p[3]),
                               Eigen::Vector2d(p[4], p[5]), Eigen::Vector2d(p[6], p[7]));
        else
            *out = cross_ratio(Eigen::Vector3d(p[0], p[1], p[2]), Eigen::Vector3d(p[3], p[4], p[5]),
                               Eigen::Vector3d(p[6], p[7], p[8]), Eigen::Vector3d(p[9], p[10], p[11]));
    });
}

int ref_require_centers_in_front(const double normal[3], double delta_min, const double* c, int32_t n) {
    return guard([&] {
        std::vector<Eigen::Vector3d> cs;
        for (int i = 0; i < n; ++i)
            cs.emplace_back(c[3 * i], c[3 * i + 1], c[3 * i + 2]);
        require_centers_in_front(Eigen::Vector3d(normal[0], normal[1], normal[2]), delta_min, cs);
    });
}

}  // extern "C"
