// K7-K9: per-pixel map kernels of the level tail (pipeline.cpp:260-301):
// winner-take-all + depth conversion + parabola refinement, the valid-only
// 5x5 median, central-difference normals, appearance-weighted normal
// smoothing with the geometric confidence fused in, and NN upscaling.
// All FP64 expression trees follow the cited reference lines; exp() is
// replaced by host-computed tables (bit-identical by construction).
// Roofline: HBM-bound map traffic (a few bytes per pixel in and out).
#include "host.hpp"
#include "kernels.hpp"

namespace fmvs {
namespace k {

namespace {

__device__ __forceinline__ double depth_from_plane_dev(double denom, double dist) {
    using namespace dev;  // geometry.cpp:299-306 with the per-pixel denominator
    if (fabs(denom) < 1e-12)
        return 0.0;
    const double d = div(-dist, denom);
    return d > 0.0 ? d : 0.0;
}

__device__ double parabola_dev(double d_prev, double d_win, double d_next, double c_prev,
                               double c_win, double c_next) {
    using namespace dev;  // sgm.cpp:351-363 (callers guarantee d_prev < d_win < d_next)
    const double num = add(add(mul(sub(mul(d_win, d_win), mul(d_next, d_next)), c_prev),
                               mul(sub(mul(d_next, d_next), mul(d_prev, d_prev)), c_win)),
                           mul(sub(mul(d_prev, d_prev), mul(d_win, d_win)), c_next));
    const double den = add(add(mul(sub(d_win, d_next), c_prev), mul(sub(d_next, d_prev), c_win)),
                           mul(sub(d_prev, d_win), c_next));
    double m = fabs(c_prev);
    if (m < fabs(c_win))
        m = fabs(c_win);
    if (m < fabs(c_next))
        m = fabs(c_next);
    if (m < 1.0)
        m = 1.0;
    if (fabs(den) < mul(1e-12, m))
        return d_win;
    const double v = div(mul(0.5, num), den);
    return v < d_prev ? d_prev : (d_next < v ? d_next : v);
}

// Winner of pixel p (plane f + best) -> winners / refined depth
// (pipeline.cpp:263-288).
__device__ __forceinline__ void wta_finish(const WtaArgs& a, int x, int y, size_t p, uint64_t e0, int f,
                                           int c, int best) {
    using namespace dev;
    const uint32_t* v32 = a.agg + e0;
    const uint16_t* v16 = reinterpret_cast<const uint16_t*>(a.agg) + e0;
    auto val = [&](int i) -> uint32_t { return a.agg16 ? v16[i] : v32[i]; };
    const int win = f + best;
    if (a.winners)
        a.winners[p] = win;
    if (!a.depth)
        return;
    const double denom = dot3(D3{a.nx, a.ny, a.nz}, unproject_px(a.intr, x, y));
    const double d_win = depth_from_plane_dev(denom, a.planes[win]);
    float out = 0.0f;
    if (d_win > 0.0) {
        double d = d_win;
        if (win - 1 >= f && win + 1 < f + c) {
            const double d_lo = depth_from_plane_dev(denom, a.planes[win + 1]);
            const double d_hi = depth_from_plane_dev(denom, a.planes[win - 1]);
            if (d_lo > 0.0 && d_hi > 0.0 && d_lo < d_win && d_win < d_hi)
                d = parabola_dev(d_lo, d_win, d_hi, double(val(best + 1)), double(val(best)),
                                 double(val(best - 1)));
        }
        out = __double2float_rn(d);
    }
    a.depth[p] = out;
}

// One thread per pixel, a sequential scan of its entries (the reference's
// first minimum): refined levels, where ranges are short.
__global__ void wta_depth_kernel(WtaArgs a) {
    using namespace dev;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= a.w)
        return;
    const size_t p = static_cast<size_t>(y) * a.w + x;
    const VolMeta m = a.meta[p];
    const int f = meta_first(m.fc), c = meta_count(m.fc);
    if (c == 0) {
        if (a.winners)
            a.winners[p] = -1;
        if (a.depth)
            a.depth[p] = 0.0f;
        return;
    }
    const uint64_t e0 = a.row_base[y] + m.rel;
    const uint32_t* v32 = a.agg + e0;
    const uint16_t* v16 = reinterpret_cast<const uint16_t*>(a.agg) + e0;
    auto val = [&](int i) -> uint32_t { return a.agg16 ? v16[i] : v32[i]; };
    int best = 0;
    uint32_t bv = val(0);
    for (int i = 1; i < c; ++i) {
        const uint32_t vi = val(i);
        if (vi < bv) {
            bv = vi;
            best = i;
        }
    }
    wta_finish(a, x, y, p, e0, f, c, best);
}

// Lane i scans entries i, i + 32, ... of one pixel (strict <: each lane's
// first minimum); (value, index) reduced with ties to the lower index.
template <typename T>
__device__ __forceinline__ int warp_argmin_first(const T* __restrict__ v, int c, int lane) {
    uint32_t bv = 0xFFFFFFFFu;
    int bi = 0x7FFFFFFF;
    for (int i = lane; i < c; i += 32) {
        const uint32_t vi = v[i];
        if (vi < bv) {
            bv = vi;
            bi = i;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const uint32_t ov = __shfl_xor_sync(0xFFFFFFFFu, bv, o);
        const int oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
        if (ov < bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
        }
    }
    return bi;
}

// Uniform (dense) levels: a warp per 32 consecutive pixels of a row; the
// warp scans each pixel's entries coalesced and finds the same first minimum
// as the sequential scan, then every lane refines its own pixel.
constexpr int kWtaWarps = 8;
__global__ void __launch_bounds__(32 * kWtaWarps) wta_depth_warp_kernel(WtaArgs a) {
    using namespace dev;
    const int lane = threadIdx.x & 31;
    const int x0 = (blockIdx.x * kWtaWarps + (threadIdx.x >> 5)) * 32;
    const int y = blockIdx.y;
    if (x0 >= a.w)
        return;  // warp-uniform
    const int x = x0 + lane;
    const bool valid = x < a.w;
    const size_t p = static_cast<size_t>(y) * a.w + x;
    int f = 0, c = 0;
    uint64_t e0 = 0;
    if (valid) {
        const VolMeta m = a.meta[p];
        f = meta_first(m.fc);
        c = meta_count(m.fc);
        e0 = a.row_base[y] + m.rel;
    }
    int best = 0;
    for (int j = 0; j < 32; ++j) {
        const int cj = __shfl_sync(0xFFFFFFFFu, c, j);
        if (cj == 0)
            continue;
        const uint64_t ej = __shfl_sync(0xFFFFFFFFu, e0, j);
        const int bj = a.agg16 ? warp_argmin_first(reinterpret_cast<const uint16_t*>(a.agg) + ej, cj, lane)
                               : warp_argmin_first(a.agg + ej, cj, lane);
        if (lane == j)
            best = bj;
    }
    if (!valid)
        return;
    if (c == 0) {
        if (a.winners)
            a.winners[p] = -1;
        if (a.depth)
            a.depth[p] = 0.0f;
        return;
    }
    wta_finish(a, x, y, p, e0, f, c, best);
}

// median_filter_5x5 (pipeline.cpp:175-198): element valid/2 of the sorted
// valid window. The 25 samples sit in registers (invalid / outside -> +inf,
// which sorts behind every valid depth), a fully unrolled Batcher odd-even
// merge network over 32 slots sorts them, and element valid/2 is picked by a
// static select chain: no local memory, no data-dependent indexing. Sorting
// only permutes values, so the result is exactly the reference's element.
// Batcher odd-even merge sorting network over 32 slots (generated).
constexpr int kMedianComparators = 191;
__device__ constexpr int8_t kMedianA[kMedianComparators] = {0,2,4,6,8,10,12,14,16,18,20,22,24,26,28,30,0,1,4,5,8,9,12,13,16,17,20,21,24,25,28,29,1,5,9,13,17,21,25,29,0,1,2,3,8,9,10,11,16,17,18,19,24,25,26,27,2,3,10,11,18,19,26,27,1,3,5,9,11,13,17,19,21,25,27,29,0,1,2,3,4,5,6,7,16,17,18,19,20,21,22,23,4,5,6,7,20,21,22,23,2,3,6,7,10,11,18,19,22,23,26,27,1,3,5,7,9,11,13,17,19,21,23,25,27,29,0,1,2,3,4,5,6,7,8,9,10,11,12,13,14,15,8,9,10,11,12,13,14,15,4,5,6,7,12,13,14,15,20,21,22,23,2,3,6,7,10,11,14,15,18,19,22,23,26,27,1,3,5,7,9,11,13,15,17,19,21,23,25,27,29};
__device__ constexpr int8_t kMedianB[kMedianComparators] = {1,3,5,7,9,11,13,15,17,19,21,23,25,27,29,31,2,3,6,7,10,11,14,15,18,19,22,23,26,27,30,31,2,6,10,14,18,22,26,30,4,5,6,7,12,13,14,15,20,21,22,23,28,29,30,31,4,5,12,13,20,21,28,29,2,4,6,10,12,14,18,20,22,26,28,30,8,9,10,11,12,13,14,15,24,25,26,27,28,29,30,31,8,9,10,11,24,25,26,27,4,5,8,9,12,13,20,21,24,25,28,29,2,4,6,8,10,12,14,18,20,22,24,26,28,30,16,17,18,19,20,21,22,23,24,25,26,27,28,29,30,31,16,17,18,19,20,21,22,23,8,9,10,11,16,17,18,19,24,25,26,27,4,5,8,9,12,13,16,17,20,21,24,25,28,29,2,4,6,8,10,12,14,16,18,20,22,24,26,28,30};

// The same network pruned for the median of 25 values (element 12): only the
// comparators that can still move a value into slot 12 (132 of the 165 that
// touch real samples), used when the whole window is valid (checked against
// full sorts of random and tied windows in tests/test_median_network.py).
constexpr int kMedian25Comparators = 132;
__device__ constexpr int8_t kMed25A[kMedian25Comparators] = {0,2,4,6,8,10,12,14,16,18,20,22,24,0,1,4,5,8,9,12,13,16,17,20,21,24,1,5,9,13,17,21,0,1,2,3,8,9,10,11,16,17,18,19,24,2,3,10,11,18,19,1,3,5,9,11,13,17,19,21,0,1,2,3,4,5,6,7,16,17,18,19,20,21,22,23,4,5,6,7,20,21,22,23,2,3,6,7,10,11,18,19,22,23,1,3,5,7,9,11,13,17,19,21,23,0,1,2,3,4,5,6,7,8,9,10,11,12,13,8,9,10,11,12,13,6,7,12,13,10,11,11};
__device__ constexpr int8_t kMed25B[kMedian25Comparators] = {1,3,5,7,9,11,13,15,17,19,21,23,25,2,3,6,7,10,11,14,15,18,19,22,23,26,2,6,10,14,18,22,4,5,6,7,12,13,14,15,20,21,22,23,28,4,5,12,13,20,21,2,4,6,10,12,14,18,20,22,8,9,10,11,12,13,14,15,24,25,26,27,28,29,30,31,8,9,10,11,24,25,26,27,4,5,8,9,12,13,20,21,24,25,2,4,6,8,10,12,14,18,20,22,24,16,17,18,19,20,21,22,23,24,25,26,27,28,29,16,17,18,19,20,21,10,11,16,17,12,13,12};

// The 5x5 window of every pixel of a 32x8 tile comes from a shared-memory copy
// of the tile + 2-pixel halo (invalid / outside samples stored as +inf); the
// window's in-image count follows from the position.
__global__ void __launch_bounds__(256) median5_kernel(const float* __restrict__ in, int w, int h,
                                                      float* __restrict__ out) {
    using namespace dev;
    constexpr int TW = 32, TH = 8, SW = TW + 4, SH = TH + 4;
    __shared__ float s_t[SH][SW];
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH;
    const int tid = threadIdx.y * TW + threadIdx.x;
    for (int r = tid; r < SW * SH; r += TW * TH) {
        const int ty = r / SW, tx = r - ty * SW;
        const int xx = x0 + tx - 2, yy = y0 + ty - 2;
        float d = INFINITY;
        if (xx >= 0 && yy >= 0 && xx < w && yy < h) {
            d = __ldg(in + static_cast<size_t>(yy) * w + xx);
            if (!depth_ok(d))
                d = INFINITY;
        }
        s_t[ty][tx] = d;
    }
    __syncthreads();
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    if (x >= w || y >= h)
        return;
    constexpr int N = 32;
    float v[N];
    int valid = 0;
#pragma unroll
    for (int dy = 0; dy < 5; ++dy)
#pragma unroll
        for (int dx = 0; dx < 5; ++dx) {
            const float d = s_t[threadIdx.y + dy][threadIdx.x + dx];
            valid += d != INFINITY ? 1 : 0;
            v[dy * 5 + dx] = d;
        }
    const int in_image = (min(x + 2, w - 1) - max(x - 2, 0) + 1) * (min(y + 2, h - 1) - max(y - 2, 0) + 1);
#pragma unroll
    for (int i = 25; i < N; ++i)
        v[i] = INFINITY;  // padding slots (both networks route through them)
    float res = 0.0f;
    if (valid == 25) {
#pragma unroll
        for (int c = 0; c < kMedian25Comparators; ++c) {
            const float lo = fminf(v[kMed25A[c]], v[kMed25B[c]]);
            const float hi = fmaxf(v[kMed25A[c]], v[kMed25B[c]]);
            v[kMed25A[c]] = lo;
            v[kMed25B[c]] = hi;
        }
        res = v[12];
    } else {
#pragma unroll
        for (int c = 0; c < kMedianComparators; ++c) {
            const float lo = fminf(v[kMedianA[c]], v[kMedianB[c]]);
            const float hi = fmaxf(v[kMedianA[c]], v[kMedianB[c]]);
            v[kMedianA[c]] = lo;
            v[kMedianB[c]] = hi;
        }
        if (!(2 * valid < in_image)) {
            const int k = valid / 2;
#pragma unroll
            for (int i = 0; i < 25; ++i)
                res = k == i ? v[i] : res;
        }
    }
    out[static_cast<size_t>(y) * w + x] = res;
}

// normals_from_depth (surface.cpp:9-39)
__global__ void normals_raw_kernel(const float* __restrict__ depth, int w, int h, dev::Intr k,
                                   float* __restrict__ out) {
    using namespace dev;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    const size_t p = static_cast<size_t>(y) * w + x;
    float3 r = make_float3(0.0f, 0.0f, 0.0f);
    if (x >= 1 && y >= 1 && x < w - 1 && y < h - 1) {
        const float dc = depth[p];
        const float dl = depth[p - 1], dr = depth[p + 1];
        const float du = depth[p - w], dd = depth[p + w];
        if (depth_ok(dc) && depth_ok(dl) && depth_ok(dr) && depth_ok(du) && depth_ok(dd)) {
            const D3 pr = scale3(double(dr), unproject_px(k, x + 1, y));
            const D3 pl = scale3(double(dl), unproject_px(k, x - 1, y));
            const D3 pd = scale3(double(dd), unproject_px(k, x, y + 1));
            const D3 pu = scale3(double(du), unproject_px(k, x, y - 1));
            const D3 hv = sub3(pr, pl);
            const D3 vv = sub3(pd, pu);
            D3 n = cross3(hv, vv);
            const double len = norm3(n);
            if (!(len < 1e-15)) {
                n = {div(n.x, len), div(n.y, len), div(n.z, len)};
                if (n.z > 0.0)
                    n = {-n.x, -n.y, -n.z};
                r = make_float3(__double2float_rn(n.x), __double2float_rn(n.y),
                                __double2float_rn(n.z));
            }
        }
    }
    out[3 * p] = r.x;
    out[3 * p + 1] = r.y;
    out[3 * p + 2] = r.z;
}

__device__ __forceinline__ float conf_of(float nx, float ny, float nz, double cos_rho,
                                         double pdv, double sx, double sy, double sz) {
    using namespace dev;  // confidence_map (surface.cpp:83-104)
    if (!normal_ok(nx, ny, nz))
        return 0.0f;
    const double ndp = dot3(D3{double(nx), double(ny), double(nz)}, D3{sx, sy, sz});
    if (ndp < cos_rho || pdv < cos_rho)
        return 0.0f;
    double score = div(sub(mul(ndp, pdv), cos_rho), sub(1.0, cos_rho));
    score = score < 0.0 ? 0.0 : (1.0 < score ? 1.0 : score);
    return __double2float_rn(score);
}

// smooth_normals (surface.cpp:41-81) + confidence_map of the smoothed normal.
// Shared-memory tiled form (radius <= 4): the 32x8 block stages its
// (32+2r)x(8+2r) window of raw normals, validity and intensities once instead
// of every thread re-loading its 5x5 neighbourhood from L1. Same arithmetic,
// same order as smooth_conf_kernel below.
constexpr int kSmMaxR = 4;
// R: the smoothing radius as a compile-time constant (1..kSmMaxR) so the
// neighbour loop unrolls and every weight / normal load is issued ahead of the
// FP64 accumulation chain; R = 0: runtime radius.
template <int R>
__global__ void smooth_conf_tiled_kernel(const float* __restrict__ raw, const uint8_t* __restrict__ img,
                                         int w, int h, int radius_rt, const double* __restrict__ wt,
                                         float* __restrict__ out, float* __restrict__ conf,
                                         double cos_rho, double pdv, double sx, double sy, double sz) {
    using namespace dev;
    const int radius = R > 0 ? R : radius_rt;
    constexpr int TW = 32 + 2 * kSmMaxR, TH = 8 + 2 * kSmMaxR;
    __shared__ float s_n[3][TH][TW];
    __shared__ int s_i[TH][TW];  // intensity, or -1 where the normal is invalid / outside
    const int bx = blockIdx.x * 32, by = blockIdx.y * 8;
    const int tw = 32 + 2 * radius, th = 8 + 2 * radius;
    for (int k = threadIdx.y * 32 + threadIdx.x; k < tw * th; k += 256) {
        const int ty = k / tw, tx = k - ty * tw;
        const int gx = bx + tx - radius, gy = by + ty - radius;
        float nx = 0.0f, ny = 0.0f, nz = 0.0f;
        int iv = -1;
        if (gx >= 0 && gy >= 0 && gx < w && gy < h) {
            const size_t q = static_cast<size_t>(gy) * w + gx;
            nx = raw[3 * q];
            ny = raw[3 * q + 1];
            nz = raw[3 * q + 2];
            if (normal_ok(nx, ny, nz))
                iv = img[q];
        }
        s_n[0][ty][tx] = nx;
        s_n[1][ty][tx] = ny;
        s_n[2][ty][tx] = nz;
        s_i[ty][tx] = iv;
    }
    __syncthreads();
    const int x = bx + threadIdx.x, y = by + threadIdx.y;
    if (x >= w || y >= h)
        return;
    const size_t p = static_cast<size_t>(y) * w + x;
    const int cx0 = threadIdx.x + radius, cy0 = threadIdx.y + radius;
    const float cx = s_n[0][cy0][cx0], cy = s_n[1][cy0][cx0], cz = s_n[2][cy0][cx0];
    float ox = 0.0f, oy = 0.0f, oz = 0.0f;
    if (s_i[cy0][cx0] >= 0) {
        double sx_ = double(cx), sy_ = double(cy), sz_ = double(cz);
        const int ic = s_i[cy0][cx0];
#pragma unroll
        for (int dy = -(R > 0 ? R : kSmMaxR); dy <= (R > 0 ? R : kSmMaxR); ++dy) {
            if (R == 0 && (dy < -radius || dy > radius))
                continue;
#pragma unroll
            for (int dx = -(R > 0 ? R : kSmMaxR); dx <= (R > 0 ? R : kSmMaxR); ++dx) {
                if (R == 0 && (dx < -radius || dx > radius))
                    continue;
                if (dx == 0 && dy == 0)
                    continue;
                const int iq = s_i[cy0 + dy][cx0 + dx];
                // outside the image or invalid normal: skipped (surface.cpp:63-67)
                // -- a select, so the sums keep the reference's exact sequence
                const bool use = iq >= 0;
                const double wq = __ldg(wt + (dx * dx + dy * dy) * 256 + (use ? abs(iq - ic) : 0));
                const double ax = add(sx_, mul(wq, double(s_n[0][cy0 + dy][cx0 + dx])));
                const double ay = add(sy_, mul(wq, double(s_n[1][cy0 + dy][cx0 + dx])));
                const double az = add(sz_, mul(wq, double(s_n[2][cy0 + dy][cx0 + dx])));
                sx_ = use ? ax : sx_;
                sy_ = use ? ay : sy_;
                sz_ = use ? az : sz_;
            }
        }
        const double len = norm3(D3{sx_, sy_, sz_});
        if (len > 1e-15) {
            ox = __double2float_rn(div(sx_, len));
            oy = __double2float_rn(div(sy_, len));
            oz = __double2float_rn(div(sz_, len));
        } else {
            ox = cx;
            oy = cy;
            oz = cz;
        }
    }
    out[3 * p] = ox;
    out[3 * p + 1] = oy;
    out[3 * p + 2] = oz;
    if (conf)
        conf[p] = conf_of(ox, oy, oz, cos_rho, pdv, sx, sy, sz);
}

__global__ void smooth_conf_kernel(const float* __restrict__ raw, const uint8_t* __restrict__ img,
                                   int w, int h, int radius, const double* __restrict__ wt,
                                   float* __restrict__ out, float* __restrict__ conf,
                                   double cos_rho, double pdv, double sx, double sy, double sz) {
    using namespace dev;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    const size_t p = static_cast<size_t>(y) * w + x;
    const float cx = raw[3 * p], cy = raw[3 * p + 1], cz = raw[3 * p + 2];
    float ox = 0.0f, oy = 0.0f, oz = 0.0f;
    if (normal_ok(cx, cy, cz)) {
        double sx_ = double(cx), sy_ = double(cy), sz_ = double(cz);
        const int ic = img[p];
        for (int dy = -radius; dy <= radius; ++dy)
            for (int dx = -radius; dx <= radius; ++dx) {
                if (dx == 0 && dy == 0)
                    continue;
                const int qx = x + dx, qy = y + dy;
                if (qx < 0 || qy < 0 || qx >= w || qy >= h)
                    continue;
                const size_t q = static_cast<size_t>(qy) * w + qx;
                const float nx = raw[3 * q], ny = raw[3 * q + 1], nz = raw[3 * q + 2];
                if (!normal_ok(nx, ny, nz))
                    continue;
                const int di = abs(int(img[q]) - ic);
                const double wq = __ldg(wt + (dx * dx + dy * dy) * 256 + di);
                sx_ = add(sx_, mul(wq, double(nx)));
                sy_ = add(sy_, mul(wq, double(ny)));
                sz_ = add(sz_, mul(wq, double(nz)));
            }
        const double len = norm3(D3{sx_, sy_, sz_});
        if (len > 1e-15) {
            ox = __double2float_rn(div(sx_, len));
            oy = __double2float_rn(div(sy_, len));
            oz = __double2float_rn(div(sz_, len));
        } else {
            ox = cx;
            oy = cy;
            oz = cz;
        }
    }
    out[3 * p] = ox;
    out[3 * p + 1] = oy;
    out[3 * p + 2] = oz;
    if (conf)
        conf[p] = conf_of(ox, oy, oz, cos_rho, pdv, sx, sy, sz);
}

__global__ void confidence_kernel(const float* __restrict__ n, int w, int h, double cos_rho,
                                  double pdv, double sx, double sy, double sz,
                                  float* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    const size_t p = static_cast<size_t>(y) * w + x;
    out[p] = conf_of(n[3 * p], n[3 * p + 1], n[3 * p + 2], cos_rho, pdv, sx, sy, sz);
}

__global__ void upscale_kernel(const float* __restrict__ in, int iw, int ih, int ch,
                               float* __restrict__ out, int ow, int oh) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= ow || y >= oh)
        return;
    const int sx = min(x / 2, iw - 1), sy = min(y / 2, ih - 1);  // pipeline.cpp:97-101
    const size_t s = static_cast<size_t>(sy) * iw + sx, d = static_cast<size_t>(y) * ow + x;
    for (int c = 0; c < ch; ++c)
        out[ch * d + c] = in[ch * s + c];
}

inline dim3 grid2(int w, int h) { return dim3((w + 31) / 32, (h + 7) / 8); }

}  // namespace

void wta_depth(const WtaArgs& a, cudaStream_t s) {
    if (a.wide)
        wta_depth_warp_kernel<<<dim3((a.w + 32 * kWtaWarps - 1) / (32 * kWtaWarps), a.h), 32 * kWtaWarps, 0,
                                s>>>(a);
    else
        wta_depth_kernel<<<dim3((a.w + 127) / 128, a.h), 128, 0, s>>>(a);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void median5(const float* in, int w, int h, float* out, cudaStream_t s) {
    median5_kernel<<<grid2(w, h), dim3(32, 8), 0, s>>>(in, w, h, out);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void normals_raw(const float* depth, int w, int h, dev::Intr intr, float* out_xyz,
                 cudaStream_t s) {
    normals_raw_kernel<<<grid2(w, h), dim3(32, 8), 0, s>>>(depth, w, h, intr, out_xyz);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void smooth_conf(const float* raw_xyz, const uint8_t* img, int w, int h, int radius,
                 const double* weights, float* out_xyz, float* conf, double cos_rho,
                 double plane_dot_view, double nx, double ny, double nz, cudaStream_t s) {
    auto tiled = [&](auto kernel) {
        kernel<<<grid2(w, h), dim3(32, 8), 0, s>>>(raw_xyz, img, w, h, radius, weights, out_xyz, conf,
                                                     cos_rho, plane_dot_view, nx, ny, nz);
    };
    if (radius == 1)
        tiled(smooth_conf_tiled_kernel<1>);
    else if (radius == 2)
        tiled(smooth_conf_tiled_kernel<2>);
    else if (radius == 3)
        tiled(smooth_conf_tiled_kernel<3>);
    else if (radius <= kSmMaxR)
        tiled(smooth_conf_tiled_kernel<0>);
    else
        smooth_conf_kernel<<<grid2(w, h), dim3(32, 8), 0, s>>>(raw_xyz, img, w, h, radius, weights,
                                                                out_xyz, conf, cos_rho,
                                                                plane_dot_view, nx, ny, nz);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void confidence(const float* normals_xyz, int w, int h, double cos_rho, double plane_dot_view,
                double nx, double ny, double nz, float* out, cudaStream_t s) {
    confidence_kernel<<<grid2(w, h), dim3(32, 8), 0, s>>>(normals_xyz, w, h, cos_rho,
                                                           plane_dot_view, nx, ny, nz, out);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void upscale(const float* in, int iw, int ih, int ch, float* out, int ow, int oh,
             cudaStream_t s) {
    upscale_kernel<<<grid2(ow, oh), dim3(32, 8), 0, s>>>(in, iw, ih, ch, out, ow, oh);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

}  // namespace k
}  // namespace fmvs
