// Host-side core of the B200 FaSS-MVS library: small fixed-size FP64 linear
// algebra, the per-level geometry the reference computes on the host
// (plane stacks, homographies, bounds), and input validation with the
// reference's error taxonomy. Everything here is data-independent, so the
// driver evaluates it for ALL levels before the first kernel launch.
//
// Numeric contract: every reduction is evaluated strictly left to right from
// the first term, with no fused multiply-add (built with -ffp-contract=off),
// which is the order the parity oracle pins (oracle/eigen_shim).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "fmvs.h"

namespace fmvs {

// Error types mapped 1:1 onto fassmvs::{InvalidInputError, ConfigError,
// GeometryError} (errors.hpp:10-24) and onto the C ABI return codes.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail_input(const std::string& m) { throw Error(FMVS_ERR_INVALID_INPUT, m); }
[[noreturn]] inline void fail_config(const std::string& m) { throw Error(FMVS_ERR_CONFIG, m); }
[[noreturn]] inline void fail_geometry(const std::string& m) { throw Error(FMVS_ERR_GEOMETRY, m); }

struct V2 {
    double x = 0, y = 0;
};
struct V3 {
    double x = 0, y = 0, z = 0;
};
struct M3 {
    double a[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // row-major
};

inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 scale(double s, V3 v) { return {s * v.x, s * v.y, s * v.z}; }
inline V3 divs(V3 v, double s) { return {v.x / s, v.y / s, v.z / s}; }
inline double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }
inline V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline V2 sub(V2 a, V2 b) { return {a.x - b.x, a.y - b.y}; }
inline double norm(V2 a) { return std::sqrt(a.x * a.x + a.y * a.y); }

inline M3 mul(const M3& p, const M3& q) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.a[i][j] = (p.a[i][0] * q.a[0][j] + p.a[i][1] * q.a[1][j]) + p.a[i][2] * q.a[2][j];
    return r;
}
inline V3 mul(const M3& m, V3 v) {
    return {(m.a[0][0] * v.x + m.a[0][1] * v.y) + m.a[0][2] * v.z,
            (m.a[1][0] * v.x + m.a[1][1] * v.y) + m.a[1][2] * v.z,
            (m.a[2][0] * v.x + m.a[2][1] * v.y) + m.a[2][2] * v.z};
}
inline M3 transpose(const M3& m) {
    M3 t;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            t.a[j][i] = m.a[i][j];
    return t;
}

struct Camera {
    fmvs_intrinsics k;
    M3 rot;
    V3 center;
};

inline Camera camera_of(const fmvs_view& v) {
    Camera c;
    c.k = v.intrinsics;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            c.rot.a[i][j] = v.pose.rotation[3 * i + j];
    c.center = {v.pose.center[0], v.pose.center[1], v.pose.center[2]};
    return c;
}
inline Camera camera_of(const fmvs_intrinsics& k, const fmvs_pose& p) {
    fmvs_view v{nullptr, k, p};
    return camera_of(v);
}

// Intrinsics::unproject (geometry.hpp:28-30).
inline V3 unproject(const fmvs_intrinsics& k, double x, double y) {
    return {(x - k.cx) / k.fx, (y - k.cy) / k.fy, 1.0};
}
// Intrinsics::halved (geometry.cpp:30-39).
inline fmvs_intrinsics halved(const fmvs_intrinsics& k) {
    return {k.fx / 2.0, k.fy / 2.0, k.cx / 2.0, k.cy / 2.0, (k.width + 1) / 2, (k.height + 1) / 2};
}

// Validation with the reference messages (geometry.cpp:17-73,
// pipeline.cpp:12-30, matching.cpp:11-18, sgm.cpp:11-20).
void validate_intrinsics(const fmvs_intrinsics& k);
void validate_pose(const M3& r);
void validate_view(const fmvs_view& v);
void validate_depth_bounds(double d_min, double d_max);
void validate_cost(const fmvs_cost_spec& c);
void validate_sgm(const fmvs_sgm_config& c);
void validate_config(const fmvs_config& c);

// Geometry (geometry.cpp:75-306).
double fractional_index(const double* d, int n, double delta);
int nearest_index(const double* d, int n, double delta);
M3 plane_homography(V3 normal, double distance, const Camera& ref, const Camera& other);
void bounding_distances(double d_min, double d_max, V3 normal, const fmvs_intrinsics& k,
                        double* delta_min, double* delta_max);
void require_centers_in_front(V3 normal, double delta_min, const std::vector<V3>& centers);
std::vector<double> plane_distances(const Camera& ref, const Camera& other, double delta_min,
                                    double delta_max, V3 normal, int max_planes);
double depth_from_plane(double x, double y, V3 normal, double distance, const fmvs_intrinsics& k);
double adaptive_phi2(double phi1, double alpha, double beta, double di);
double parabola_refine(double d_prev, double d_win, double d_next, double c_prev, double c_win,
                       double c_next);

// Host-computed lookup tables replacing every transcendental on the path.
std::vector<long long> phi2_table(const fmvs_sgm_config& cfg);          // 256 entries
std::vector<double> smoothing_table(int radius);                         // (2r^2+1) x 256
void blur3_kernel(double k[3]);                                          // sigma 1, radius 1
std::vector<double> blur_kernel(int radius, double sigma);               // pipeline.cpp:33-40
std::vector<uint16_t> census_cost_table(int bits);                       // bits+1 entries

}  // namespace fmvs
