// Device-side primitives shared by the sm_100a kernels.
//
// Parity contract: every FP64 operation that feeds an
// integer result (census bits, NCC cost, plane intervals, SGM shifts) is an
// explicit IEEE round-to-nearest intrinsic (__dadd_rn/__dmul_rn/__ddiv_rn/
// __dsqrt_rn), never contracted into an FMA (the library is also built with
// --fmad=false), in the reference's expression order.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "fmvs.h"

namespace fmvs {
namespace dev {

// Camera intrinsics as passed to kernels.
struct Intr {
    double fx, fy, cx, cy;
    int w, h;
    // optional per-level unprojection tables (device): ux[x + 1] =
    // (x - cx) / fx for x in [-1, w], uy[y + 1] likewise -- the exact values
    // of unproject's two divisions, built on the host (IEEE division)
    const double* ux = nullptr;
    const double* uy = nullptr;
};
inline Intr make_intr(const fmvs_intrinsics& k) { return {k.fx, k.fy, k.cx, k.cy, k.width, k.height}; }

// Ragged cost-volume layout in HBM:
//   meta[p] = {offset of pixel p relative to its row base,
//              first | count << 16}
//   row_base[y] = entry index of the row's first hypothesis (u64)
struct VolMeta {
    uint32_t rel;
    uint32_t fc;
};

#ifdef __CUDACC__
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }

struct D3 {
    double x, y, z;
};

__device__ __forceinline__ double dot3(D3 a, D3 b) {
    return add(add(mul(a.x, b.x), mul(a.y, b.y)), mul(a.z, b.z));
}
__device__ __forceinline__ D3 scale3(double s, D3 v) { return {mul(s, v.x), mul(s, v.y), mul(s, v.z)}; }
__device__ __forceinline__ D3 sub3(D3 a, D3 b) { return {sub(a.x, b.x), sub(a.y, b.y), sub(a.z, b.z)}; }
__device__ __forceinline__ D3 add3(D3 a, D3 b) { return {add(a.x, b.x), add(a.y, b.y), add(a.z, b.z)}; }
__device__ __forceinline__ D3 cross3(D3 a, D3 b) {
    return {sub(mul(a.y, b.z), mul(a.z, b.y)), sub(mul(a.z, b.x), mul(a.x, b.z)),
            sub(mul(a.x, b.y), mul(a.y, b.x))};
}
__device__ __forceinline__ double norm3(D3 a) { return sqrt_(dot3(a, a)); }

// Intrinsics::unproject (geometry.hpp:28-30).
__device__ __forceinline__ D3 unproject(const Intr& k, double x, double y) {
    return {div(sub(x, k.cx), k.fx), div(sub(y, k.cy), k.fy), 1.0};
}
// unproject of an integer pixel, from the tables when the level has them
__device__ __forceinline__ D3 unproject_px(const Intr& k, int x, int y) {
    if (k.ux && static_cast<unsigned>(x + 1) <= static_cast<unsigned>(k.w + 1) &&
        static_cast<unsigned>(y + 1) <= static_cast<unsigned>(k.h + 1))
        return {k.ux[x + 1], k.uy[y + 1], 1.0};
    return unproject(k, double(x), double(y));
}

// float validity predicates (raster.hpp:64-65), evaluated in float.
__device__ __forceinline__ bool depth_ok(float d) { return d > 0.0f && isfinite(d); }
__device__ __forceinline__ bool normal_ok(float x, float y, float z) {
    return __fadd_rn(__fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y)), __fmul_rn(z, z)) > 0.0f;
}

// PlaneStack::fractional_index / nearest_index (geometry.cpp:75-98).
__device__ __forceinline__ double fractional_index(const double* d, int n, double delta) {
    if (n <= 1)
        return 0.0;
    if (delta >= d[0])
        return div(-sub(delta, d[0]), sub(d[0], d[1]));
    if (delta <= d[n - 1])
        return add(double(n - 1), div(sub(d[n - 1], delta), sub(d[n - 2], d[n - 1])));
    int lo = 0, hi = n - 1;
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (d[mid] >= delta)
            lo = mid;
        else
            hi = mid;
    }
    return add(double(lo), div(sub(d[lo], delta), sub(d[lo], d[lo + 1])));
}

__device__ __forceinline__ int nearest_index(const double* d, int n, double delta) {
    const double f = fractional_index(d, n, delta);
    const int i = static_cast<int>(llround(f));
    return i < 0 ? 0 : (i > n - 1 ? n - 1 : i);
}

__device__ __forceinline__ int meta_first(uint32_t fc) { return int(fc & 0xFFFFu); }
__device__ __forceinline__ int meta_count(uint32_t fc) { return int(fc >> 16); }
#endif  // __CUDACC__

}  // namespace dev
}  // namespace fmvs

#define FMVS_CUDA_CHECK(expr)                                                           \
    do {                                                                                \
        cudaError_t fmvs_e_ = (expr);                                                   \
        if (fmvs_e_ != cudaSuccess)                                                     \
            throw ::fmvs::Error(FMVS_ERR_CUDA, std::string(#expr) + ": " +              \
                                                   cudaGetErrorString(fmvs_e_));         \
    } while (0)
