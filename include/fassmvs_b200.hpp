// fassmvs_b200.hpp -- header-only C++ adapter from the reference's public C++
// API (proj/include/fassmvs/*.hpp) to the B200 library's C ABI (fmvs.h).
//
// Include AFTER the reference headers are on the include path (they bring
// Eigen and the fassmvs types). Every function keeps the reference
// signature and error behaviour: C-ABI return codes are rethrown as
// fassmvs::InvalidInputError / ConfigError / GeometryError
// (errors.hpp:10-24); device failures as std::runtime_error.
//
//   fassmvs_b200::estimate_bundle(bundle, config)   // pipeline.hpp:79-80
//
// Defining FASSMVS_B200_DEFINE_ESTIMATE_BUNDLE in exactly one translation
// unit additionally defines fassmvs::estimate_bundle itself on top of the
// B200 library -- the drop-in used by INTEGRATION.md (the reference's CPU
// definition is compiled under another name with
// -Destimate_bundle=estimate_bundle_cpu on pipeline.cpp only).
// FASSMVS_B200_DEFINE_POSTFILTER does the same for dog_mask and
// geometric_consistency_mask (postfilter.cpp compiled with the two names
// renamed).
#pragma once

#include <algorithm>
#include <array>
#include <cstring>
#include <span>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fassmvs/colorize.hpp"
#include "fassmvs/errors.hpp"
#include "fassmvs/map_io.hpp"
#include "fassmvs/matching.hpp"
#include "fassmvs/pipeline.hpp"
#include "fassmvs/postfilter.hpp"
#include "fassmvs/sgm.hpp"
#include "fassmvs/surface.hpp"
#include "fmvs.h"

namespace fassmvs_b200 {

inline void check(int rc) {
    if (rc == FMVS_OK)
        return;
    const std::string msg = fmvs_last_error();
    switch (rc) {
        case FMVS_ERR_INVALID_INPUT:
            throw fassmvs::InvalidInputError(msg);
        case FMVS_ERR_CONFIG:
            throw fassmvs::ConfigError(msg);
        case FMVS_ERR_GEOMETRY:
            throw fassmvs::GeometryError(msg);
        default:
            throw std::runtime_error("fassmvs_b200: " + msg);
    }
}

// One CUDA context/stream + device arenas. Not reentrant; one per thread.
class Context {
public:
    explicit Context(int device = 0) { check(fmvs_ctx_create(device, &ctx_)); }
    ~Context() { fmvs_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    fmvs_ctx* get() const { return ctx_; }

    // Per-thread default context on the calling thread's current CUDA device
    // (cudaSetDevice before the call picks the GPU; one context per thread
    // and device). The reference's functions are free functions safe to call
    // concurrently (README.md:160-162), so a multi-threaded caller spreads
    // bundles over GPUs by setting a device per thread.
    static Context& thread_default() {
        thread_local std::vector<std::unique_ptr<Context>> per_device;
        const int dev = fmvs_current_device();
        if (dev < 0)
            check(FMVS_ERR_CUDA);
        if (static_cast<size_t>(dev) >= per_device.size())
            per_device.resize(dev + 1);
        if (!per_device[dev])
            per_device[dev] = std::make_unique<Context>(dev);
        return *per_device[dev];
    }

private:
    fmvs_ctx* ctx_ = nullptr;
};

inline fmvs_intrinsics to_c(const fassmvs::Intrinsics& k) {
    return {k.fx, k.fy, k.cx, k.cy, k.width, k.height};
}

inline fmvs_pose to_c(const fassmvs::Pose& p) {
    fmvs_pose r{};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.rotation[3 * i + j] = p.rotation(i, j);
    for (int i = 0; i < 3; ++i)
        r.center[i] = p.center(i);
    return r;
}

inline fmvs_sgm_config to_c(const fassmvs::SgmConfig& s) {
    return {static_cast<int32_t>(s.variant), s.paths, s.phi1, s.phi2_adaptive ? 1 : 0,
            s.phi2_fixed, s.alpha, s.beta, s.penalty_scale};
}

inline fmvs_config to_c(const fassmvs::PipelineConfig& p) {
    fmvs_config c{};
    c.bundle_size = p.bundle_size;
    c.pyramid_levels = p.pyramid_levels;
    c.d_min = p.depth_bounds.d_min;
    c.d_max = p.depth_bounds.d_max;
    for (int i = 0; i < 3; ++i)
        c.sweep_normal[i] = p.sweep_normal(i);
    c.range_kind = static_cast<int32_t>(p.range_policy.kind);
    c.range_value = p.range_policy.value;
    c.max_planes = p.max_planes;
    c.sgm = to_c(p.sgm);
    c.cost = {static_cast<int32_t>(p.cost.kind), p.cost.window_w, p.cost.window_h};
    c.normal_smoothing_radius = p.normal_smoothing_radius;
    return c;
}

inline std::vector<fmvs_view> to_c(const std::vector<fassmvs::CalibratedView>& bundle) {
    std::vector<fmvs_view> v(bundle.size());
    for (size_t k = 0; k < bundle.size(); ++k) {
        // image size must match the intrinsics (geometry.cpp:56-61); the C
        // ABI carries one size, so the mismatch is rejected here.
        const auto& b = bundle[k];
        if (b.image.width() != b.intrinsics.width || b.image.height() != b.intrinsics.height)
            throw fassmvs::InvalidInputError("calibrated view: image size does not match intrinsics");
        v[k] = fmvs_view{b.image.data(), to_c(b.intrinsics), to_c(b.pose)};
    }
    return v;
}

// fassmvs::estimate_bundle (pipeline.hpp:79-80) on the B200 library.
inline fassmvs::BundleResult estimate_bundle(const std::vector<fassmvs::CalibratedView>& bundle,
                                             const fassmvs::PipelineConfig& config,
                                             Context& ctx = Context::thread_default()) {
    const std::vector<fmvs_view> views = to_c(bundle);
    const fmvs_config cfg = to_c(config);
    const int w = bundle.empty() ? 1 : std::max(1, bundle[bundle.size() / 2].intrinsics.width);
    const int h = bundle.empty() ? 1 : std::max(1, bundle[bundle.size() / 2].intrinsics.height);
    fassmvs::BundleResult r;
    r.depth = fassmvs::DepthMap(w, h, 0.0f);
    r.confidence = fassmvs::ConfidenceMap(w, h, 0.0f);
    std::vector<float> normals(static_cast<size_t>(w) * h * 3);
    check(fmvs_estimate_bundle(ctx.get(), views.data(), static_cast<int32_t>(views.size()), &cfg,
                               r.depth.data(), normals.data(), r.confidence.data()));
    r.normals = fassmvs::make_normal_map(w, h);
    for (size_t p = 0; p < static_cast<size_t>(w) * h; ++p)
        r.normals.data()[p] = Eigen::Vector3f(normals[3 * p], normals[3 * p + 1], normals[3 * p + 2]);
    return r;
}

// fassmvs::sweep_cost_volume (matching.hpp:74-76) on the B200 library.
inline fassmvs::CostVolume sweep_cost_volume(const std::vector<fassmvs::CalibratedView>& bundle,
                                             int ref_index, const fassmvs::PlaneStack& planes,
                                             const fassmvs::SamplingRange& ranges,
                                             const fassmvs::CostFunctionSpec& costfn,
                                             Context& ctx = Context::thread_default()) {
    const std::vector<fmvs_view> views = to_c(bundle);
    fmvs_plane_stack ps{{planes.normal(0), planes.normal(1), planes.normal(2)},
                        planes.distances.data(), planes.count()};
    const fmvs_cost_spec cs{static_cast<int32_t>(costfn.kind), costfn.window_w, costfn.window_h};
    fassmvs::CostVolume v;
    v.width = ranges.lo.width();
    v.height = ranges.lo.height();
    v.planes = planes;
    const size_t npx = static_cast<size_t>(v.width) * v.height;
    v.first.resize(npx);
    v.count.resize(npx);
    std::vector<uint64_t> off(npx);
    uint64_t total = 0;
    int32_t per_side = 0;
    uint64_t cap = npx * static_cast<uint64_t>(std::max(1, planes.count()));
    v.costs.resize(cap);
    check(fmvs_sweep_cost_volume(ctx.get(), views.data(), static_cast<int32_t>(views.size()),
                                 ref_index, &ps, ranges.lo.data(), ranges.hi.data(), &cs,
                                 v.first.data(), v.count.data(), off.data(), v.costs.data(), cap,
                                 &total, &per_side));
    v.costs.resize(total);
    v.offset.assign(off.begin(), off.end());
    v.per_side = per_side;
    return v;
}


// ------------------------------------------------------------------ stages
// The stage-level public functions of the reference API on the
// B200 library, each with the reference signature and error behaviour.

inline fmvs_plane_stack to_c(const fassmvs::PlaneStack& p) {
    return fmvs_plane_stack{{p.normal(0), p.normal(1), p.normal(2)}, p.distances.data(), p.count()};
}

inline std::vector<float> normals_xyz(const fassmvs::NormalMap& m) {
    std::vector<float> out(3 * m.size());
    for (size_t p = 0; p < m.size(); ++p) {
        out[3 * p] = m.data()[p].x();
        out[3 * p + 1] = m.data()[p].y();
        out[3 * p + 2] = m.data()[p].z();
    }
    return out;
}

inline fassmvs::NormalMap normal_map(const std::vector<float>& xyz, int w, int h) {
    fassmvs::NormalMap m = fassmvs::make_normal_map(w, h);
    for (size_t p = 0; p < static_cast<size_t>(w) * h; ++p)
        m.data()[p] = Eigen::Vector3f(xyz[3 * p], xyz[3 * p + 1], xyz[3 * p + 2]);
    return m;
}

// build_pyramids (pipeline.hpp:50, pipeline.cpp:107-126).
inline fassmvs::PyramidLevelSet build_pyramids(const std::vector<fassmvs::CalibratedView>& bundle,
                                               int levels, Context& ctx = Context::thread_default()) {
    if (levels < 1)
        throw fassmvs::ConfigError("pyramids: need at least one level");
    for (const auto& v : bundle)
        v.validate();
    const std::vector<fmvs_view> views = to_c(bundle);
    const int n = static_cast<int>(views.size());
    // level sizes: ceil-halving of every view (Intrinsics::halved, geometry.cpp:30-39)
    uint64_t cap = 0;
    for (const auto& v : bundle) {
        fassmvs::Intrinsics k = v.intrinsics;
        for (int l = 0; l < levels; ++l, k = k.halved())
            cap += static_cast<uint64_t>(k.width) * k.height;
    }
    std::vector<uint8_t> images(std::max<uint64_t>(cap, 1));
    std::vector<fmvs_intrinsics> intr(static_cast<size_t>(levels) * n);
    check(fmvs_build_pyramids(ctx.get(), views.data(), n, levels, images.data(), cap, intr.data()));
    fassmvs::PyramidLevelSet set;
    set.levels.resize(levels);
    size_t o = 0;
    for (int l = 0; l < levels; ++l)
        for (int k = 0; k < n; ++k) {
            const fmvs_intrinsics& c = intr[static_cast<size_t>(l) * n + k];
            fassmvs::CalibratedView v;
            v.intrinsics = fassmvs::Intrinsics{c.fx, c.fy, c.cx, c.cy, c.width, c.height};
            v.pose = bundle[k].pose;
            v.image = fassmvs::ImageU8(c.width, c.height, 0);
            std::memcpy(v.image.data(), images.data() + o, static_cast<size_t>(c.width) * c.height);
            o += static_cast<size_t>(c.width) * c.height;
            set.levels[l].push_back(std::move(v));
        }
    return set;
}

// gaussian_blur (pipeline.hpp:54, pipeline.cpp:32-75).
inline fassmvs::Raster<float> gaussian_blur(const fassmvs::ImageU8& image, int radius, double sigma,
                                            Context& ctx = Context::thread_default()) {
    fassmvs::Raster<float> out(image.width(), image.height(), 0.0f);
    check(fmvs_gaussian_blur(ctx.get(), image.data(), image.width(), image.height(), radius, sigma,
                             out.data()));
    return out;
}

// upscale_nearest (pipeline.hpp:58-59, pipeline.cpp:91-134).
inline fassmvs::DepthMap upscale_nearest(const fassmvs::DepthMap& map, int width, int height,
                                         Context& ctx = Context::thread_default()) {
    if (width == map.width() && height == map.height())
        return map;
    fassmvs::DepthMap out(std::max(width, 0), std::max(height, 0), 0.0f);
    check(fmvs_upscale_nearest(ctx.get(), map.data(), map.width(), map.height(), 1, width, height,
                               out.data()));
    return out;
}

inline fassmvs::NormalMap upscale_nearest(const fassmvs::NormalMap& map, int width, int height,
                                          Context& ctx = Context::thread_default()) {
    if (width == map.width() && height == map.height())
        return map;
    const std::vector<float> in = normals_xyz(map);
    std::vector<float> out(3 * static_cast<size_t>(std::max(width, 0)) * std::max(height, 0));
    check(fmvs_upscale_nearest(ctx.get(), in.data(), map.width(), map.height(), 3, width, height,
                               out.data()));
    return normal_map(out, width, height);
}

// refine_range (pipeline.hpp:63-65, pipeline.cpp:136-173).
inline fassmvs::SamplingRange refine_range(const fassmvs::DepthMap& prior,
                                           const fassmvs::RangePolicy& policy,
                                           const fassmvs::DepthBounds& bounds,
                                           const fassmvs::PlaneStack* coarser_planes = nullptr,
                                           const fassmvs::Intrinsics* intrinsics = nullptr,
                                           Context& ctx = Context::thread_default()) {
    fassmvs::SamplingRange r;
    r.lo = fassmvs::Raster<float>(prior.width(), prior.height(), 0.0f);
    r.hi = fassmvs::Raster<float>(prior.width(), prior.height(), 0.0f);
    const fmvs_plane_stack ps = coarser_planes ? to_c(*coarser_planes) : fmvs_plane_stack{};
    const fmvs_intrinsics in = intrinsics ? to_c(*intrinsics) : fmvs_intrinsics{};
    check(fmvs_refine_range(ctx.get(), prior.data(), prior.width(), prior.height(),
                            static_cast<int32_t>(policy.kind), policy.value, bounds.d_min, bounds.d_max,
                            coarser_planes ? &ps : nullptr, intrinsics ? &in : nullptr, r.lo.data(),
                            r.hi.data()));
    return r;
}

// median_filter_5x5 (pipeline.hpp:72, pipeline.cpp:175-198).
inline fassmvs::DepthMap median_filter_5x5(const fassmvs::DepthMap& depth,
                                           Context& ctx = Context::thread_default()) {
    fassmvs::DepthMap out(depth.width(), depth.height(), 0.0f);
    check(fmvs_median_filter_5x5(ctx.get(), depth.data(), depth.width(), depth.height(), out.data()));
    return out;
}

// census_transform (matching.hpp:58, matching.cpp:44-55).
inline fassmvs::Raster<std::uint64_t> census_transform(const fassmvs::ImageU8& image, int window_w,
                                                       int window_h,
                                                       Context& ctx = Context::thread_default()) {
    fassmvs::Raster<std::uint64_t> out(image.width(), image.height(), 0);
    check(fmvs_census_transform(ctx.get(), image.data(), image.width(), image.height(), window_w,
                                window_h, reinterpret_cast<uint64_t*>(out.data())));
    return out;
}

// census_bits_at (matching.hpp:60) and ncc_cost (matching.hpp:64): host.
inline std::uint64_t census_bits_at(const fassmvs::ImageU8& image, int x, int y, int window_w,
                                    int window_h) {
    return fmvs_census_bits_at(image.data(), image.width(), image.height(), x, y, window_w, window_h);
}

inline int ncc_cost(std::span<const float> a, std::span<const float> b) {
    if (a.size() != b.size() || a.empty())
        throw fassmvs::InvalidInputError("ncc: patches must be non-empty and equal size");
    int32_t cost = 0;
    check(fmvs_ncc_cost(a.data(), b.data(), static_cast<int32_t>(a.size()), &cost));
    return cost;
}

// compute_normal_offsets (sgm.hpp:66-68, sgm.cpp:252-299).
inline fassmvs::NormalOffsets compute_normal_offsets(const fassmvs::NormalMap& prior_normals,
                                                     const fassmvs::DepthMap& prior_depth,
                                                     const fassmvs::PlaneStack& planes,
                                                     const fassmvs::Intrinsics& intrinsics,
                                                     Context& ctx = Context::thread_default()) {
    if (!prior_normals.same_size(prior_depth))
        throw fassmvs::InvalidInputError("normal offsets: normal and depth map sizes differ");
    const int w = prior_normals.width(), h = prior_normals.height();
    fassmvs::NormalOffsets out(w, h, std::array<std::int16_t, 4>{0, 0, 0, 0});
    const std::vector<float> n = normals_xyz(prior_normals);
    const fmvs_plane_stack ps = to_c(planes);
    const fmvs_intrinsics in = to_c(intrinsics);
    static_assert(sizeof(std::array<std::int16_t, 4>) == 8, "packed shifts");
    check(fmvs_compute_normal_offsets(ctx.get(), n.data(), prior_depth.data(), w, h, &ps, &in,
                                      reinterpret_cast<int16_t*>(out.data())));
    return out;
}

namespace detail {

// aggregate / aggregate_single_path on the C ABI; `all` selects every
// config.paths direction.
inline fassmvs::AggregatedVolume aggregate(const fassmvs::CostVolume& vol, const fassmvs::ImageU8& image,
                                           const fassmvs::SgmConfig& config,
                                           const fassmvs::Intrinsics& intrinsics, bool all, int dx,
                                           int dy, const fassmvs::NormalMap* prior_normals,
                                           const fassmvs::DepthMap* prior_depth, Context& ctx) {
    // check_aggregate_inputs (sgm.cpp:241-248), then the offsets' size check
    config.validate();
    if (image.width() != vol.width || image.height() != vol.height)
        throw fassmvs::InvalidInputError("sgm: image size does not match the cost volume");
    const bool sn = config.variant == fassmvs::SgmVariant::SurfaceNormal;
    if (sn && (!prior_normals || !prior_depth))
        throw fassmvs::ConfigError("sgm: surface-normal variant requires a prior normal and depth map");
    if (sn && !prior_normals->same_size(*prior_depth))
        throw fassmvs::InvalidInputError("normal offsets: normal and depth map sizes differ");
    if (sn && (prior_depth->width() != vol.width || prior_depth->height() != vol.height))
        throw fassmvs::InvalidInputError("sgm: prior maps must match the cost volume size");
    fassmvs::AggregatedVolume agg;
    agg.width = vol.width;
    agg.height = vol.height;
    agg.planes = vol.planes;
    agg.first = vol.first;
    agg.count = vol.count;
    agg.offset = vol.offset;
    agg.values.assign(vol.costs.size(), 0);
    const std::vector<uint64_t> off(vol.offset.begin(), vol.offset.end());
    const fmvs_plane_stack ps = to_c(vol.planes);
    const fmvs_sgm_config sc = to_c(config);
    const fmvs_intrinsics in = to_c(intrinsics);
    std::vector<float> pn;
    if (sn)
        pn = normals_xyz(*prior_normals);
    const float* pd = sn ? prior_depth->data() : nullptr;
    if (all)
        check(fmvs_aggregate(ctx.get(), vol.width, vol.height, &ps, vol.first.data(), vol.count.data(),
                             off.data(), vol.costs.data(), vol.costs.size(), image.data(), &sc, &in,
                             sn ? pn.data() : nullptr, pd, 0, 0, agg.values.data()));
    else
        check(fmvs_aggregate_single_path(ctx.get(), vol.width, vol.height, &ps, vol.first.data(),
                                         vol.count.data(), off.data(), vol.costs.data(), vol.costs.size(),
                                         image.data(), &sc, &in, sn ? pn.data() : nullptr, pd, dx, dy,
                                         agg.values.data()));
    return agg;
}

}  // namespace detail

// aggregate (sgm.hpp:83-86, sgm.cpp:317-331).
inline fassmvs::AggregatedVolume aggregate(const fassmvs::CostVolume& volume, const fassmvs::ImageU8& image,
                                           const fassmvs::SgmConfig& config,
                                           const fassmvs::Intrinsics& intrinsics,
                                           const fassmvs::NormalMap* prior_normals = nullptr,
                                           const fassmvs::DepthMap* prior_depth = nullptr,
                                           Context& ctx = Context::thread_default()) {
    return detail::aggregate(volume, image, config, intrinsics, true, 0, 0, prior_normals, prior_depth, ctx);
}

// aggregate_single_path (sgm.hpp:88-92, sgm.cpp:301-315): any integer step.
inline fassmvs::AggregatedVolume aggregate_single_path(const fassmvs::CostVolume& volume,
                                                       const fassmvs::ImageU8& image,
                                                       const fassmvs::SgmConfig& config,
                                                       const fassmvs::Intrinsics& intrinsics, int dir_x,
                                                       int dir_y,
                                                       const fassmvs::NormalMap* prior_normals = nullptr,
                                                       const fassmvs::DepthMap* prior_depth = nullptr,
                                                       Context& ctx = Context::thread_default()) {
    return detail::aggregate(volume, image, config, intrinsics, false, dir_x, dir_y, prior_normals,
                             prior_depth, ctx);
}

// wta (sgm.hpp:95, sgm.cpp:333-349).
inline fassmvs::PlaneIndexMap wta(const fassmvs::AggregatedVolume& volume,
                                  Context& ctx = Context::thread_default()) {
    fassmvs::PlaneIndexMap map(volume.width, volume.height, -1);
    const std::vector<uint64_t> off(volume.offset.begin(), volume.offset.end());
    check(fmvs_wta(ctx.get(), volume.width, volume.height, volume.first.data(), volume.count.data(),
                   off.data(), volume.values.data(), volume.values.size(), map.data()));
    return map;
}

// adaptive_phi2 (sgm.hpp:36) and parabola_refine (sgm.hpp:100-101): host.
inline double adaptive_phi2(double phi1, double alpha, double beta, double intensity_delta) {
    return fmvs_adaptive_phi2(phi1, alpha, beta, intensity_delta);
}

inline double parabola_refine(double d_prev, double d_win, double d_next, double c_prev, double c_win,
                              double c_next) {
    double out = 0.0;
    check(fmvs_parabola_refine(d_prev, d_win, d_next, c_prev, c_win, c_next, &out));
    return out;
}

// normals_from_depth / smooth_normals / confidence_map (surface.hpp:11-24).
inline fassmvs::NormalMap normals_from_depth(const fassmvs::DepthMap& depth,
                                             const fassmvs::Intrinsics& intrinsics,
                                             Context& ctx = Context::thread_default()) {
    std::vector<float> out(3 * depth.size());
    const fmvs_intrinsics in = to_c(intrinsics);
    check(fmvs_normals_from_depth(ctx.get(), depth.data(), depth.width(), depth.height(), &in, out.data()));
    return normal_map(out, depth.width(), depth.height());
}

inline fassmvs::NormalMap smooth_normals(const fassmvs::NormalMap& raw, const fassmvs::ImageU8& image,
                                         int radius, Context& ctx = Context::thread_default()) {
    if (!raw.same_size(image))
        throw fassmvs::InvalidInputError("smooth normals: image size differs");
    const std::vector<float> in = normals_xyz(raw);
    std::vector<float> out(in.size());
    check(fmvs_smooth_normals(ctx.get(), in.data(), image.data(), raw.width(), raw.height(), radius,
                              out.data()));
    return normal_map(out, raw.width(), raw.height());
}

inline fassmvs::ConfidenceMap confidence_map(const fassmvs::NormalMap& normals,
                                             const Eigen::Vector3d& sweep_normal, double rho_degrees = 60.0,
                                             Context& ctx = Context::thread_default()) {
    const std::vector<float> in = normals_xyz(normals);
    fassmvs::ConfidenceMap out(normals.width(), normals.height(), 0.0f);
    const double n[3] = {sweep_normal(0), sweep_normal(1), sweep_normal(2)};
    check(fmvs_confidence_map(ctx.get(), in.data(), normals.width(), normals.height(), n, rho_degrees,
                              out.data()));
    return out;
}

// ------------------------------------------------------ host geometry
// (geometry.hpp:98-140) on the library's host restatement.

inline Eigen::Matrix3d plane_homography(const fassmvs::SweepPlane& plane, const fassmvs::Intrinsics& ref_intr,
                                        const fassmvs::Pose& ref_pose, const fassmvs::Intrinsics& other_intr,
                                        const fassmvs::Pose& other_pose) {
    const double n[3] = {plane.normal(0), plane.normal(1), plane.normal(2)};
    const fmvs_intrinsics ri = to_c(ref_intr), oi = to_c(other_intr);
    const fmvs_pose rp = to_c(ref_pose), op = to_c(other_pose);
    double h[9];
    check(fmvs_plane_homography(n, plane.distance, &ri, &rp, &oi, &op, h));
    Eigen::Matrix3d m;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            m(r, c) = h[3 * r + c];
    return m;
}

inline Eigen::Vector2d apply_homography(const Eigen::Matrix3d& h, const Eigen::Vector2d& px) {
    double hm[9], out[2];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            hm[3 * r + c] = h(r, c);
    fmvs_apply_homography(hm, px.x(), px.y(), out);
    return Eigen::Vector2d(out[0], out[1]);
}

inline std::pair<double, double> bounding_distances(const fassmvs::DepthBounds& bounds,
                                                    const Eigen::Vector3d& normal,
                                                    const fassmvs::Intrinsics& ref_intr) {
    const double n[3] = {normal(0), normal(1), normal(2)};
    const fmvs_intrinsics ri = to_c(ref_intr);
    double lo = 0.0, hi = 0.0;
    check(fmvs_bounding_distances(bounds.d_min, bounds.d_max, n, &ri, &lo, &hi));
    return {lo, hi};
}

inline void require_centers_in_front(const Eigen::Vector3d& normal, double delta_min,
                                     std::span<const Eigen::Vector3d> centers_in_ref) {
    const double n[3] = {normal(0), normal(1), normal(2)};
    std::vector<double> c(3 * centers_in_ref.size());
    for (size_t i = 0; i < centers_in_ref.size(); ++i)
        for (int j = 0; j < 3; ++j)
            c[3 * i + j] = centers_in_ref[i](j);
    check(fmvs_require_centers_in_front(n, delta_min, c.data(), static_cast<int32_t>(centers_in_ref.size())));
}

inline double cross_ratio(const Eigen::Vector2d& p1, const Eigen::Vector2d& p2, const Eigen::Vector2d& p3,
                          const Eigen::Vector2d& p4) {
    const double p[8] = {p1.x(), p1.y(), p2.x(), p2.y(), p3.x(), p3.y(), p4.x(), p4.y()};
    double out = 0.0;
    check(fmvs_cross_ratio(p, 2, &out));
    return out;
}

inline double cross_ratio(const Eigen::Vector3d& p1, const Eigen::Vector3d& p2, const Eigen::Vector3d& p3,
                          const Eigen::Vector3d& p4) {
    const double p[12] = {p1.x(), p1.y(), p1.z(), p2.x(), p2.y(), p2.z(),
                          p3.x(), p3.y(), p3.z(), p4.x(), p4.y(), p4.z()};
    double out = 0.0;
    check(fmvs_cross_ratio(p, 3, &out));
    return out;
}

inline std::vector<double> plane_distances(const fassmvs::Intrinsics& ref_intr, const fassmvs::Pose& ref_pose,
                                           const fassmvs::Intrinsics& other_intr,
                                           const fassmvs::Pose& other_pose, double delta_min,
                                           double delta_max, const Eigen::Vector3d& normal, int max_planes) {
    const double n[3] = {normal(0), normal(1), normal(2)};
    const fmvs_intrinsics ri = to_c(ref_intr), oi = to_c(other_intr);
    const fmvs_pose rp = to_c(ref_pose), op = to_c(other_pose);
    int32_t count = 0;
    std::vector<double> out(1024);
    int rc = fmvs_plane_distances(&ri, &rp, &oi, &op, delta_min, delta_max, n, max_planes, out.data(),
                                  static_cast<int32_t>(out.size()), &count);
    if (rc == FMVS_ERR_CAPACITY) {
        out.resize(count);
        rc = fmvs_plane_distances(&ri, &rp, &oi, &op, delta_min, delta_max, n, max_planes, out.data(),
                                  count, &count);
    }
    check(rc);
    out.resize(count);
    return out;
}

inline double depth_from_plane(const Eigen::Vector2d& pixel, const fassmvs::SweepPlane& plane,
                               const fassmvs::Intrinsics& intr) {
    const double n[3] = {plane.normal(0), plane.normal(1), plane.normal(2)};
    const fmvs_intrinsics in = to_c(intr);
    return fmvs_depth_from_plane(pixel.x(), pixel.y(), n, plane.distance, &in);
}

// fassmvs::dog_mask (postfilter.hpp:18) on the B200 library.
inline fassmvs::TextureMask dog_mask(const fassmvs::ImageU8& image,
                                     Context& ctx = Context::thread_default()) {
    fassmvs::TextureMask m(image.width(), image.height(), 0);
    check(fmvs_dog_mask(ctx.get(), image.data(), image.width(), image.height(), m.data()));
    return m;
}

// fassmvs::geometric_consistency_mask (postfilter.hpp:44-45) on the B200 library.
inline fassmvs::TextureMask geometric_consistency_mask(
    const std::vector<fassmvs::ConsistencyView>& window, int ref_index,
    const fassmvs::GeomFilterConfig& config = {}, Context& ctx = Context::thread_default()) {
    std::vector<fmvs_consistency_view> w(window.size());
    for (size_t k = 0; k < window.size(); ++k)
        w[k] = fmvs_consistency_view{window[k].depth.data(), window[k].depth.width(),
                                     window[k].depth.height(), to_c(window[k].intrinsics),
                                     to_c(window[k].pose)};
    const fmvs_geom_filter_config c{config.eta_r, config.eta_h,
                                    config.lookup == fassmvs::DepthLookup::Bilinear ? FMVS_LOOKUP_BILINEAR
                                                                                    : FMVS_LOOKUP_NEAREST};
    const bool ok = ref_index >= 0 && ref_index < static_cast<int>(window.size());
    fassmvs::TextureMask keep(ok ? window[ref_index].depth.width() : 0,
                              ok ? window[ref_index].depth.height() : 0, 1);
    check(fmvs_geometric_consistency_mask(ctx.get(), w.data(), static_cast<int32_t>(w.size()),
                                          ref_index, &c, keep.data()));
    return keep;
}

// Output stage of the CLI (colorize.hpp:9-15, map_io.hpp:25-27).
inline fassmvs::RgbImage rgb_image(const std::vector<std::uint8_t>& rgb, int w, int h) {
    fassmvs::RgbImage img(w, h);
    for (size_t i = 0; i < img.size(); ++i)
        img.data()[i] = {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
    return img;
}
inline fassmvs::RgbImage colorize_depth(const fassmvs::DepthMap& map, double lo, double hi,
                                        Context& ctx = Context::thread_default()) {
    std::vector<std::uint8_t> rgb(3 * map.size());
    check(fmvs_colorize_depth(ctx.get(), map.data(), map.width(), map.height(), lo, hi, rgb.data()));
    return rgb_image(rgb, map.width(), map.height());
}
inline fassmvs::RgbImage colorize_normals(const fassmvs::NormalMap& map, Context& ctx = Context::thread_default()) {
    const std::vector<float> xyz = normals_xyz(map);
    std::vector<std::uint8_t> rgb(3 * map.size());
    check(fmvs_colorize_normals(ctx.get(), xyz.data(), map.width(), map.height(), rgb.data()));
    return rgb_image(rgb, map.width(), map.height());
}
inline fassmvs::RgbImage colorize_confidence(const fassmvs::ConfidenceMap& map,
                                             Context& ctx = Context::thread_default()) {
    std::vector<std::uint8_t> rgb(3 * map.size());
    check(fmvs_colorize_confidence(ctx.get(), map.data(), map.width(), map.height(), rgb.data()));
    return rgb_image(rgb, map.width(), map.height());
}
inline void write_pfm(const std::string& path, const fassmvs::DepthMap& map) {
    check(fmvs_write_pfm(path.c_str(), map.data(), map.width(), map.height(), 1));
}
inline void write_pfm(const std::string& path, const fassmvs::NormalMap& map) {
    const std::vector<float> xyz = normals_xyz(map);
    check(fmvs_write_pfm(path.c_str(), xyz.data(), map.width(), map.height(), 3));
}
inline void write_png(const std::string& path, const fassmvs::RgbImage& image) {
    std::vector<std::uint8_t> rgb(3 * image.size());
    for (size_t i = 0; i < image.size(); ++i)
        for (int c = 0; c < 3; ++c)
            rgb[3 * i + c] = image.data()[i][c];
    check(fmvs_write_png(path.c_str(), rgb.data(), image.width(), image.height()));
}

}  // namespace fassmvs_b200

#ifdef FASSMVS_B200_DEFINE_ESTIMATE_BUNDLE
namespace fassmvs {
// The drop-in: the reference's entry point, served by the B200 library.
BundleResult estimate_bundle(const std::vector<CalibratedView>& bundle, const PipelineConfig& config) {
    return fassmvs_b200::estimate_bundle(bundle, config);
}
}  // namespace fassmvs
#endif

#ifdef FASSMVS_B200_DEFINE_POSTFILTER
namespace fassmvs {
// The post-filter entry points (postfilter.hpp:18,44-45) served by the B200
// library (postfilter.cpp compiled with -Ddog_mask=dog_mask_cpu
// -Dgeometric_consistency_mask=geometric_consistency_mask_cpu).
TextureMask dog_mask(const ImageU8& image) { return fassmvs_b200::dog_mask(image); }
TextureMask geometric_consistency_mask(const std::vector<ConsistencyView>& window, int ref_index,
                                       const GeomFilterConfig& config) {
    return fassmvs_b200::geometric_consistency_mask(window, ref_index, config);
}
}  // namespace fassmvs
#endif

#ifdef FASSMVS_B200_DEFINE_STAGES
namespace fassmvs {
// The stage-level entry points (pipeline.hpp:50-72, matching.hpp:58-76,
// sgm.hpp:36-101, surface.hpp:11-24, geometry.hpp:98-140) served by the B200
// library; the reference sources defining them are compiled with each name
// renamed (oracle/Makefile).
PyramidLevelSet build_pyramids(const std::vector<CalibratedView>& bundle, int levels) {
    return fassmvs_b200::build_pyramids(bundle, levels);
}
Raster<float> gaussian_blur(const ImageU8& image, int radius, double sigma) {
    return fassmvs_b200::gaussian_blur(image, radius, sigma);
}
DepthMap upscale_nearest(const DepthMap& map, int width, int height) {
    return fassmvs_b200::upscale_nearest(map, width, height);
}
NormalMap upscale_nearest(const NormalMap& map, int width, int height) {
    return fassmvs_b200::upscale_nearest(map, width, height);
}
SamplingRange refine_range(const DepthMap& prior, const RangePolicy& policy, const DepthBounds& bounds,
                           const PlaneStack* coarser_planes, const Intrinsics* intrinsics) {
    return fassmvs_b200::refine_range(prior, policy, bounds, coarser_planes, intrinsics);
}
DepthMap median_filter_5x5(const DepthMap& depth) { return fassmvs_b200::median_filter_5x5(depth); }
Raster<std::uint64_t> census_transform(const ImageU8& image, int window_w, int window_h) {
    return fassmvs_b200::census_transform(image, window_w, window_h);
}
std::uint64_t census_bits_at(const ImageU8& image, int x, int y, int window_w, int window_h) {
    return fassmvs_b200::census_bits_at(image, x, y, window_w, window_h);
}
int ncc_cost(std::span<const float> patch_ref, std::span<const float> patch_other) {
    return fassmvs_b200::ncc_cost(patch_ref, patch_other);
}
CostVolume sweep_cost_volume(const std::vector<CalibratedView>& bundle, int ref_index,
                             const PlaneStack& planes, const SamplingRange& ranges,
                             const CostFunctionSpec& costfn) {
    return fassmvs_b200::sweep_cost_volume(bundle, ref_index, planes, ranges, costfn);
}
NormalOffsets compute_normal_offsets(const NormalMap& prior_normals, const DepthMap& prior_depth,
                                     const PlaneStack& planes, const Intrinsics& intrinsics) {
    return fassmvs_b200::compute_normal_offsets(prior_normals, prior_depth, planes, intrinsics);
}
AggregatedVolume aggregate(const CostVolume& volume, const ImageU8& image, const SgmConfig& config,
                           const Intrinsics& intrinsics, const NormalMap* prior_normals,
                           const DepthMap* prior_depth) {
    return fassmvs_b200::aggregate(volume, image, config, intrinsics, prior_normals, prior_depth);
}
AggregatedVolume aggregate_single_path(const CostVolume& volume, const ImageU8& image,
                                       const SgmConfig& config, const Intrinsics& intrinsics, int dir_x,
                                       int dir_y, const NormalMap* prior_normals, const DepthMap* prior_depth) {
    return fassmvs_b200::aggregate_single_path(volume, image, config, intrinsics, dir_x, dir_y, prior_normals,
                                               prior_depth);
}
PlaneIndexMap wta(const AggregatedVolume& volume) { return fassmvs_b200::wta(volume); }
double adaptive_phi2(double phi1, double alpha, double beta, double intensity_delta) {
    return fassmvs_b200::adaptive_phi2(phi1, alpha, beta, intensity_delta);
}
double parabola_refine(double d_prev, double d_win, double d_next, double c_prev, double c_win,
                       double c_next) {
    return fassmvs_b200::parabola_refine(d_prev, d_win, d_next, c_prev, c_win, c_next);
}
NormalMap normals_from_depth(const DepthMap& depth, const Intrinsics& intrinsics) {
    return fassmvs_b200::normals_from_depth(depth, intrinsics);
}
NormalMap smooth_normals(const NormalMap& raw, const ImageU8& image, int radius) {
    return fassmvs_b200::smooth_normals(raw, image, radius);
}
ConfidenceMap confidence_map(const NormalMap& normals, const Eigen::Vector3d& sweep_normal, double rho_degrees) {
    return fassmvs_b200::confidence_map(normals, sweep_normal, rho_degrees);
}
Eigen::Matrix3d plane_homography(const SweepPlane& plane, const Intrinsics& ref_intr, const Pose& ref_pose,
                                 const Intrinsics& other_intr, const Pose& other_pose) {
    return fassmvs_b200::plane_homography(plane, ref_intr, ref_pose, other_intr, other_pose);
}
Eigen::Vector2d apply_homography(const Eigen::Matrix3d& h, const Eigen::Vector2d& px) {
    return fassmvs_b200::apply_homography(h, px);
}
std::pair<double, double> bounding_distances(const DepthBounds& bounds, const Eigen::Vector3d& normal,
                                             const Intrinsics& ref_intr) {
    return fassmvs_b200::bounding_distances(bounds, normal, ref_intr);
}
void require_centers_in_front(const Eigen::Vector3d& normal, double delta_min,
                              std::span<const Eigen::Vector3d> centers_in_ref) {
    fassmvs_b200::require_centers_in_front(normal, delta_min, centers_in_ref);
}
double cross_ratio(const Eigen::Vector2d& p1, const Eigen::Vector2d& p2, const Eigen::Vector2d& p3,
                   const Eigen::Vector2d& p4) {
    return fassmvs_b200::cross_ratio(p1, p2, p3, p4);
}
double cross_ratio(const Eigen::Vector3d& p1, const Eigen::Vector3d& p2, const Eigen::Vector3d& p3,
                   const Eigen::Vector3d& p4) {
    return fassmvs_b200::cross_ratio(p1, p2, p3, p4);
}
std::vector<double> plane_distances(const Intrinsics& ref_intr, const Pose& ref_pose, const Intrinsics& other_intr,
                                    const Pose& other_pose, double delta_min, double delta_max,
                                    const Eigen::Vector3d& normal, int max_planes) {
    return fassmvs_b200::plane_distances(ref_intr, ref_pose, other_intr, other_pose, delta_min, delta_max,
                                         normal, max_planes);
}
double depth_from_plane(const Eigen::Vector2d& pixel, const SweepPlane& plane, const Intrinsics& intr) {
    return fassmvs_b200::depth_from_plane(pixel, plane, intr);
}
}  // namespace fassmvs
#endif

#ifdef FASSMVS_B200_DEFINE_OUTPUT
namespace fassmvs {
// The CLI's output stage (colorize.hpp:9-15, map_io.hpp:25-27) served by the
// B200 library (colorize.cpp / map_io.cpp compiled with each name renamed
// <name>_cpu, oracle/Makefile).
RgbImage colorize_depth(const DepthMap& map, double lo, double hi) {
    return fassmvs_b200::colorize_depth(map, lo, hi);
}
RgbImage colorize_normals(const NormalMap& map) { return fassmvs_b200::colorize_normals(map); }
RgbImage colorize_confidence(const ConfidenceMap& map) { return fassmvs_b200::colorize_confidence(map); }
void write_pfm(const std::string& path, const DepthMap& map) { fassmvs_b200::write_pfm(path, map); }
void write_pfm(const std::string& path, const NormalMap& map) { fassmvs_b200::write_pfm(path, map); }
void write_png(const std::string& path, const RgbImage& image) { fassmvs_b200::write_png(path, image); }
}  // namespace fassmvs
#endif
