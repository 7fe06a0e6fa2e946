// Host geometry and validation. Each function restates the cited reference
// function with the same floating-point expression trees (see host.hpp).
#include <algorithm>
#include <cmath>
#include <limits>

#include "host.hpp"

namespace fmvs {

namespace {
constexpr double kOrthoTol = 1e-9;    // geometry.cpp:11
constexpr double kUnitTol = 1e-9;     // geometry.cpp:12
constexpr double kParallel = 1e-12;   // geometry.cpp:13

M3 intrinsic_matrix(const fmvs_intrinsics& k) {
    M3 m;
    m.a[0][0] = k.fx;
    m.a[0][2] = k.cx;
    m.a[1][1] = k.fy;
    m.a[1][2] = k.cy;
    m.a[2][2] = 1;
    return m;
}

// Unsigned sine of the angle between two rays (geometry.cpp:167-169).
double ray_sine(V3 a, V3 b) { return norm(cross(a, b)) / (norm(a) * norm(b)); }

V2 project(const fmvs_intrinsics& k, V3 p) {
    return {k.fx * p.x / p.z + k.cx, k.fy * p.y / p.z + k.cy};
}
}  // namespace

// ------------------------------------------------------------ validation --

void validate_intrinsics(const fmvs_intrinsics& k) {  // geometry.cpp:17-22
    if (!(k.fx > 0.0) || !(k.fy > 0.0))
        fail_input("intrinsics: focal lengths must be positive");
    if (k.width < 1 || k.height < 1)
        fail_input("intrinsics: image dimensions must be at least 1");
}

void validate_pose(const M3& r) {  // geometry.cpp:41-47
    const M3 gram = mul(r, transpose(r));
    double worst = 0.0;
    bool first = true;
    for (int j = 0; j < 3; ++j)  // column-major scan like Eigen's maxCoeff
        for (int i = 0; i < 3; ++i) {
            const double e = std::abs(gram.a[i][j] - (i == j ? 1.0 : 0.0));
            if (first || e > worst) {
                worst = e;
                first = false;
            }
        }
    if (worst > kOrthoTol)
        fail_input("pose: rotation is not orthonormal");
    const auto h = [&](int a, int b, int c) {
        return r.a[0][a] * (r.a[1][b] * r.a[2][c] - r.a[1][c] * r.a[2][b]);
    };
    const double det = h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1);
    if (std::abs(det - 1.0) > kOrthoTol)
        fail_input("pose: rotation determinant is not +1");
}

void validate_view(const fmvs_view& v) {  // geometry.cpp:56-61
    validate_intrinsics(v.intrinsics);
    validate_pose(camera_of(v).rot);
    if (v.image == nullptr)
        fail_input("calibrated view: image size does not match intrinsics");
}

void validate_depth_bounds(double d_min, double d_max) {  // geometry.cpp:70-73
    if (!(d_min > 0.0) || !(d_min < d_max))
        fail_input("depth bounds: need 0 < d_min < d_max");
}

void validate_cost(const fmvs_cost_spec& c) {  // matching.cpp:11-18
    const bool census_ok = c.kind == FMVS_COST_CENSUS &&
                           ((c.window_w == 5 && c.window_h == 5) || (c.window_w == 9 && c.window_h == 7));
    const bool ncc_ok = c.kind == FMVS_COST_NCC &&
                        ((c.window_w == 5 && c.window_h == 5) || (c.window_w == 9 && c.window_h == 9));
    if (!census_ok && !ncc_ok)
        fail_config("cost function: unsupported window size");
}

void validate_sgm(const fmvs_sgm_config& c) {  // sgm.cpp:11-20
    if (c.paths != 8 && c.paths != 4)
        fail_config("sgm: paths must be 8 or 4");
    if (c.phi1 < 0.0)
        fail_config("sgm: penalties must be non-negative");
    if (!c.phi2_adaptive && c.phi2_fixed < c.phi1)
        fail_config("sgm: the second penalty must not be smaller than the first");
    if (c.penalty_scale < 1)
        fail_config("sgm: penalty scale must be at least 1");
    if (c.variant < FMVS_SGM_PLANE || c.variant > FMVS_SGM_PATH_GRADIENT)
        fail_config("sgm: unknown variant");
}

void validate_config(const fmvs_config& c) {  // pipeline.cpp:12-30
    if (c.bundle_size < 3 || c.bundle_size % 2 == 0)
        fail_config("pipeline: bundle size must be odd and at least 3");
    if (c.pyramid_levels < 1)
        fail_config("pipeline: need at least one pyramid level");
    validate_depth_bounds(c.d_min, c.d_max);
    const V3 n{c.sweep_normal[0], c.sweep_normal[1], c.sweep_normal[2]};
    if (std::abs(norm(n) - 1.0) > 1e-9)
        fail_config("pipeline: sweep normal must be unit length");
    if (c.max_planes < 2)
        fail_config("pipeline: max_planes must be at least 2");
    if (c.normal_smoothing_radius < 1)
        fail_config("pipeline: normal smoothing radius must be at least 1");
    validate_sgm(c.sgm);
    validate_cost(c.cost);
    if (c.range_kind < FMVS_RANGE_FULL || c.range_kind > FMVS_RANGE_SPACING_MULTIPLE)
        fail_config("pipeline: unknown range policy");
    if (c.sgm.variant == FMVS_SGM_SURFACE_NORMAL && c.pyramid_levels < 2)
        fail_config(
            "pipeline: surface-normal SGM needs a prior normal map and therefore at least "
            "two pyramid levels");
}

// -------------------------------------------------------------- geometry --

// PlaneStack::fractional_index (geometry.cpp:75-93): same bisection.
double fractional_index(const double* d, int n, double delta) {
    if (n <= 1)
        return 0.0;
    if (delta >= d[0])
        return -(delta - d[0]) / (d[0] - d[1]);
    if (delta <= d[n - 1])
        return (n - 1) + (d[n - 1] - delta) / (d[n - 2] - d[n - 1]);
    int lo = 0, hi = n - 1;
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (d[mid] >= delta)
            lo = mid;
        else
            hi = mid;
    }
    return lo + (d[lo] - delta) / (d[lo] - d[lo + 1]);
}

int nearest_index(const double* d, int n, double delta) {  // geometry.cpp:95-98
    const double f = fractional_index(d, n, delta);
    return std::clamp(static_cast<int>(std::llround(f)), 0, n - 1);
}

// K_o (R_o R_ref^T - t n^T / delta) K_ref^-1 (geometry.cpp:100-114).
M3 plane_homography(V3 normal, double distance, const Camera& ref, const Camera& other) {
    if (std::abs(norm(normal) - 1.0) > kUnitTol)
        fail_input("sweep plane: normal must be unit length");
    if (!(distance > 0.0))
        fail_input("sweep plane: distance must be positive");
    validate_intrinsics(ref.k);
    validate_intrinsics(other.k);
    const M3 r = mul(other.rot, transpose(ref.rot));
    const V3 t = mul(other.rot, sub(ref.center, other.center));
    const double tv[3] = {t.x, t.y, t.z};
    const double nv[3] = {normal.x, normal.y, normal.z};
    M3 mid;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            mid.a[i][j] = r.a[i][j] - (tv[i] * nv[j]) / distance;
    M3 kinv;
    kinv.a[0][0] = 1.0 / ref.k.fx;
    kinv.a[0][2] = -ref.k.cx / ref.k.fx;
    kinv.a[1][1] = 1.0 / ref.k.fy;
    kinv.a[1][2] = -ref.k.cy / ref.k.fy;
    kinv.a[2][2] = 1;
    return mul(mul(intrinsic_matrix(other.k), mid), kinv);
}

// Frustum-corner bounding distances (geometry.cpp:121-145).
void bounding_distances(double d_min, double d_max, V3 normal, const fmvs_intrinsics& k,
                        double* delta_min, double* delta_max) {
    validate_depth_bounds(d_min, d_max);
    validate_intrinsics(k);
    if (std::abs(norm(normal) - 1.0) > kUnitTol)
        fail_input("bounding distances: normal must be unit length");
    const double cx[4] = {0.0, double(k.width - 1), 0.0, double(k.width - 1)};
    const double cy[4] = {0.0, 0.0, double(k.height - 1), double(k.height - 1)};
    double lo = std::numeric_limits<double>::infinity();
    double hi = std::numeric_limits<double>::infinity();
    for (int c = 0; c < 4; ++c) {
        const V3 ray = unproject(k, cx[c], cy[c]);
        lo = std::min(lo, std::abs(dot(normal, scale(d_min, ray))));
        hi = std::min(hi, std::abs(dot(normal, scale(d_max, ray))));
    }
    if (!(lo > 0.0) || !(lo < hi))
        fail_geometry("bounding distances: sweep normal degenerate for this frustum");
    *delta_min = lo;
    *delta_max = hi;
}

void require_centers_in_front(V3 normal, double delta_min, const std::vector<V3>& centers) {
    for (const V3& c : centers)  // geometry.cpp:147-153
        if (!(dot(normal, c) + delta_min > 0.0))
            fail_geometry("sweep geometry: camera center behind the near bounding plane");
}

// Unit-pixel plane spacing by the cross-ratio along the epipolar segment of
// the extremal corner (geometry.cpp:183-297).
std::vector<double> plane_distances(const Camera& ref, const Camera& other, double delta_min,
                                    double delta_max, V3 normal, int max_planes) {
    if (!(delta_min > 0.0) || delta_min > delta_max)
        fail_input("plane distances: need 0 < delta_min <= delta_max");
    if (max_planes < 1)
        fail_config("plane distances: max_planes must be at least 1");
    if (delta_min == delta_max)
        return {delta_min};

    const M3 h_near = plane_homography(normal, delta_min, ref, other);
    const double cxs[4] = {0.0, double(ref.k.width - 1), 0.0, double(ref.k.width - 1)};
    const double cys[4] = {0.0, 0.0, double(ref.k.height - 1), double(ref.k.height - 1)};
    V2 p_ref{cxs[0], cys[0]};
    double best = -1.0;
    for (int c = 0; c < 4; ++c) {
        const V3 q = mul(h_near, V3{cxs[c], cys[c], 1.0});
        const V2 warped{q.x / q.z, q.y / q.z};
        const double disp = norm(sub(warped, V2{cxs[c], cys[c]}));
        if (disp > best) {
            best = disp;
            p_ref = {cxs[c], cys[c]};
        }
    }

    const V3 ray = unproject(ref.k, p_ref.x, p_ref.y);
    const double denom = dot(normal, ray);
    if (std::abs(denom) < kParallel)
        fail_geometry("plane distances: corner ray parallel to the sweep planes");
    const V3 p_min_ref = scale(-delta_min / denom, ray);
    const V3 p_max_ref = scale(-delta_max / denom, ray);

    const M3 rel_rot = mul(other.rot, transpose(ref.rot));
    const V3 rel_t = mul(other.rot, sub(ref.center, other.center));
    const V3 v_epipole = rel_t;
    if (norm(v_epipole) < kParallel)
        fail_geometry("plane distances: zero baseline between the two cameras");

    const V3 x_min = add(mul(rel_rot, p_min_ref), rel_t);
    const V3 x_max = add(mul(rel_rot, p_max_ref), rel_t);
    if (!(x_min.z > 0.0) || !(x_max.z > 0.0))
        fail_geometry("plane distances: bounding intersections behind the other camera");
    const V2 px_min = project(other.k, x_min);
    const V2 px_max = project(other.k, x_max);

    const double span = norm(sub(px_min, px_max));
    if (span < kParallel)
        fail_geometry("plane distances: no disparity change across the depth range");
    if (span > 1e6)
        fail_geometry("plane distances: epipolar segment degenerate (near epipole)");
    const V2 step{(px_min.x - px_max.x) / span, (px_min.y - px_max.y) / span};

    const V3 v_max = unproject(other.k, px_max.x, px_max.y);
    const V3 v_min = unproject(other.k, px_min.x, px_min.y);
    const double sin_e_max = ray_sine(v_epipole, v_max);
    const double sin_min_max = ray_sine(v_min, v_max);
    if (sin_e_max < kParallel || sin_min_max < kParallel)
        fail_geometry("plane distances: epipole coincides with a bounding point");

    std::vector<double> out;
    out.reserve(static_cast<std::size_t>(span) + 2);
    out.push_back(delta_max);
    const double range = delta_max - delta_min;
    for (double t = 1.0; t < span; t += 1.0) {
        const V2 px{px_max.x + t * step.x, px_max.y + t * step.y};
        const V3 v = unproject(other.k, px.x, px.y);
        const double sin_e_i = ray_sine(v_epipole, v);
        const double sin_min_i = ray_sine(v_min, v);
        if (sin_min_i < kParallel)
            break;
        const double q = (sin_e_i * sin_min_max) / (sin_e_max * sin_min_i);
        const double denom_q = q * delta_max - range;
        if (!(denom_q > 0.0))
            fail_geometry("plane distances: cross-ratio solve degenerate");
        const double delta = q * delta_max * delta_min / denom_q;
        if (delta <= delta_min || delta >= out.back())
            continue;
        out.push_back(delta);
    }
    out.push_back(delta_min);

    const int n = static_cast<int>(out.size());
    if (n <= max_planes)
        return out;
    std::vector<double> picked;
    picked.reserve(max_planes);
    for (int m = 0; m < max_planes; ++m) {
        const int idx =
            static_cast<int>(std::llround(static_cast<double>(m) * (n - 1) / (max_planes - 1)));
        if (picked.empty() || out[idx] < picked.back())
            picked.push_back(out[idx]);
    }
    return picked;
}

double depth_from_plane(double x, double y, V3 normal, double distance,
                        const fmvs_intrinsics& k) {  // geometry.cpp:299-306
    const double denom = dot(normal, unproject(k, x, y));
    if (std::abs(denom) < kParallel)
        return 0.0;
    const double d = -distance / denom;
    return d > 0.0 ? d : 0.0;
}

double adaptive_phi2(double phi1, double alpha, double beta, double di) {  // sgm.cpp:22-24
    return phi1 * (1.0 + alpha * std::exp(-di / beta));
}

double parabola_refine(double d_prev, double d_win, double d_next, double c_prev, double c_win,
                       double c_next) {  // sgm.cpp:351-363
    if (!(d_prev < d_win && d_win < d_next))
        fail_input("parabola refine: depths must be strictly increasing");
    const double num = (d_win * d_win - d_next * d_next) * c_prev +
                       (d_next * d_next - d_prev * d_prev) * c_win +
                       (d_prev * d_prev - d_win * d_win) * c_next;
    const double den = (d_win - d_next) * c_prev + (d_next - d_prev) * c_win +
                       (d_prev - d_win) * c_next;
    if (std::abs(den) <
        1e-12 * std::max({std::abs(c_prev), std::abs(c_win), std::abs(c_next), 1.0}))
        return d_win;
    return std::clamp(0.5 * num / den, d_prev, d_next);
}

// --------------------------------------------------------------- tables --

std::vector<long long> phi2_table(const fmvs_sgm_config& cfg) {  // sgm.cpp:118-126
    std::vector<long long> t(256);
    for (int di = 0; di < 256; ++di)
        t[di] = cfg.phi2_adaptive
                    ? std::llround(adaptive_phi2(cfg.phi1, cfg.alpha, cfg.beta, double(di)) *
                                   cfg.penalty_scale)
                    : std::llround(cfg.phi2_fixed * cfg.penalty_scale);
    return t;
}

// gauss_norm * exp(-dist2 / (2 sigma^2) - di / beta), sigma = radius, beta = 10
// (surface.cpp:48-49, 71-72), indexed [dist2][di].
std::vector<double> smoothing_table(int radius) {
    const double sigma = radius;
    const double beta = 10.0;
    const double gauss_norm = 1.0 / std::sqrt(2.0 * M_PI * sigma * sigma);
    const int nd = 2 * radius * radius + 1;
    std::vector<double> t(static_cast<std::size_t>(nd) * 256);
    for (int d2 = 0; d2 < nd; ++d2)
        for (int di = 0; di < 256; ++di) {
            const double dist2 = static_cast<double>(d2);
            const double dd = static_cast<double>(di);
            t[static_cast<std::size_t>(d2) * 256 + di] =
                gauss_norm * std::exp(-dist2 / (2.0 * sigma * sigma) - dd / beta);
        }
    return t;
}

std::vector<double> blur_kernel(int radius, double sigma) {  // pipeline.cpp:33-40
    std::vector<double> k(2 * radius + 1);
    double sum = 0.0;
    for (int i = -radius; i <= radius; ++i) {
        k[i + radius] = std::exp(-0.5 * i * i / (sigma * sigma));
        sum += k[i + radius];
    }
    for (auto& v : k)
        v /= sum;
    return k;
}

void blur3_kernel(double k[3]) {  // gaussian_blur(radius 1, sigma 1), pipeline.cpp:33-40
    const int radius = 1;
    const double sigma = 1.0;
    double sum = 0.0;
    for (int i = -radius; i <= radius; ++i) {
        k[i + radius] = std::exp(-0.5 * i * i / (sigma * sigma));
        sum += k[i + radius];
    }
    for (int i = 0; i < 3; ++i)
        k[i] /= sum;
}

std::vector<uint16_t> census_cost_table(int bits) {  // matching.cpp:259-260
    std::vector<uint16_t> t(bits + 1);
    for (int ham = 0; ham <= bits; ++ham)
        t[ham] = static_cast<uint16_t>(std::lround(255.0 * ham / bits));
    return t;
}

}  // namespace fmvs
