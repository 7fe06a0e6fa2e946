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

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fassmvs/errors.hpp"
#include "fassmvs/matching.hpp"
#include "fassmvs/pipeline.hpp"
#include "fassmvs/postfilter.hpp"
#include "fassmvs/sgm.hpp"
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

    // Per-thread default context on device 0 (the reference's functions are
    // free functions safe to call concurrently, README.md:160-162).
    static Context& thread_default() {
        thread_local std::unique_ptr<Context> c;
        if (!c)
            c = std::make_unique<Context>(0);
        return *c;
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
