// K4: plane-sweep multi-image matching into the dynamic cost volume
// (sweep_cost_volume, matching.cpp:116-294; Alg. 1 of the paper).
//
// Mapping: one CTA per 32-pixel row segment. A segment's hypotheses are
// contiguous in the ragged volume, so the CTA flattens (pixel, plane) into
// one index space and its threads stride over it (load-balanced across the
// ragged per-pixel counts). Each thread evaluates one hypothesis over all
// matching views: homography centre, inside test, window walk with the
// reference's sequential column increments, FP64 bilinear samples from the
// quad-packed image (one 32-bit load = the four taps), census Hamming or
// NCC, per-side sums and min(left, right) -> u16.
//
// Bit-exactness: the FP64 path follows matching.cpp:222-281 operation by
// operation (IEEE intrinsics, no FMA). The census centre sample is taken
// first (same sequential walk) so the window need not be stored.
// Roofline: FP64-issue-bound (~50 DP ops per bilinear sample); HBM traffic is
// 2 B per hypothesis written plus the (L2-resident) images.
#include <algorithm>
#include <type_traits>


#include "host.hpp"
#include "kernels.hpp"

namespace fmvs {
namespace k {

namespace {

constexpr int kSeg = 32;
constexpr int kThreads = 128;

struct Hom {
    double h[9];
};

// bilinear() of raster.hpp:71-84 on a quad-packed image, with the caller's
// perspective divide (matching.cpp:242-244).
__device__ __forceinline__ double warp_sample(const uint32_t* __restrict__ quad, int w, int h,
                                              double qx, double qy, double qz) {
    using namespace dev;
    if (!(qz > 0.0))
        return 0.0;
    double x = div(qx, qz);
    double y = div(qy, qz);
    const double xm = double(w - 1), ym = double(h - 1);
    x = x < 0.0 ? 0.0 : (xm < x ? xm : x);  // std::clamp
    y = y < 0.0 ? 0.0 : (ym < y ? ym : y);
    const int x0 = __double2int_rz(x);
    const int y0 = __double2int_rz(y);
    const uint32_t q = __ldg(quad + static_cast<size_t>(y0) * w + x0);
    const double ax = sub(x, double(x0));
    const double ay = sub(y, double(y0));
    const double omx = sub(1.0, ax);
    const double top = add(mul(omx, double(q & 0xFFu)), mul(ax, double((q >> 8) & 0xFFu)));
    const double bot = add(mul(omx, double((q >> 16) & 0xFFu)), mul(ax, double(q >> 24)));
    return add(mul(sub(1.0, ay), top), mul(ay, bot));
}

template <int KIND, int WW, int WH>
__device__ __forceinline__ int view_cost(const uint32_t* __restrict__ quad, int vw, int vh,
                                         const double* __restrict__ hp, double xd, double yd,
                                         uint64_t ref_bits, const float* __restrict__ ref_patch,
                                         double ref_mean, double ref_var,
                                         const uint16_t* __restrict__ lut) {
    using namespace dev;
    constexpr int RX = WW / 2, RY = WH / 2, NS = WW * WH;
    double H[9];
#pragma unroll
    for (int i = 0; i < 9; ++i)
        H[i] = __ldg(hp + i);
    // center = hom * (x, y, 1) (matching.cpp:222-223); H(i,2) * 1.0 is exact.
    const double cx = add(add(mul(H[0], xd), mul(H[1], yd)), H[2]);
    const double cy = add(add(mul(H[3], xd), mul(H[4], yd)), H[5]);
    const double cz = add(add(mul(H[6], xd), mul(H[7], yd)), H[8]);
    bool inside = false;
    if (cz > 0.0) {
        const double cxw = div(cx, cz), cyw = div(cy, cz);
        inside = cxw >= 0.0 && cyw >= 0.0 && cxw <= double(vw) - 1.0 && cyw <= double(vh) - 1.0;
    }
    if (!inside)
        return 255;
    // row_start = center - rx * step_x - ry * step_y (matching.cpp:238)
    double rsx = sub(sub(cx, mul(double(RX), H[0])), mul(double(RY), H[1]));
    double rsy = sub(sub(cy, mul(double(RX), H[3])), mul(double(RY), H[4]));
    double rsz = sub(sub(cz, mul(double(RX), H[6])), mul(double(RY), H[7]));
    if constexpr (KIND == FMVS_COST_CENSUS) {
        // Centre sample first, reached by the same sequential increments.
        double qx = rsx, qy = rsy, qz = rsz;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            qx = add(qx, H[1]);
            qy = add(qy, H[4]);
            qz = add(qz, H[7]);
        }
#pragma unroll
        for (int c = 0; c < RX; ++c) {
            qx = add(qx, H[0]);
            qy = add(qy, H[3]);
            qz = add(qz, H[6]);
        }
        const double wc = warp_sample(quad, vw, vh, qx, qy, qz);
        uint64_t bits = 0;
#pragma unroll
        for (int r = 0; r < WH; ++r) {
            qx = rsx;
            qy = rsy;
            qz = rsz;
#pragma unroll
            for (int c = 0; c < WW; ++c) {
                if (!(r == RY && c == RX)) {
                    const double v = warp_sample(quad, vw, vh, qx, qy, qz);
                    bits = (bits << 1) | (v < wc ? 1u : 0u);
                }
                qx = add(qx, H[0]);
                qy = add(qy, H[3]);
                qz = add(qz, H[6]);
            }
            rsx = add(rsx, H[1]);
            rsy = add(rsy, H[4]);
            rsz = add(rsz, H[7]);
        }
        return lut[__popcll(bits ^ ref_bits)];
    } else {
        if (ref_var <= 0.0)
            return 255;
        double sb = 0.0, sbb = 0.0, sab = 0.0;
        int s = 0;
#pragma unroll
        for (int r = 0; r < WH; ++r) {
            double qx = rsx, qy = rsy, qz = rsz;
#pragma unroll
            for (int c = 0; c < WW; ++c) {
                const double v = warp_sample(quad, vw, vh, qx, qy, qz);
                sb = add(sb, v);
                sbb = add(sbb, mul(v, v));
                sab = add(sab, mul(double(ref_patch[s]), v));
                ++s;
                qx = add(qx, H[0]);
                qy = add(qy, H[3]);
                qz = add(qz, H[6]);
            }
            rsx = add(rsx, H[1]);
            rsy = add(rsy, H[4]);
            rsz = add(rsz, H[7]);
        }
        const double var_b = sub(sbb, div(mul(sb, sb), double(NS)));
        if (var_b <= 0.0)
            return 255;
        const double ncc = div(sub(sab, mul(ref_mean, sb)), sqrt_(mul(ref_var, var_b)));
        const double t = sub(1.0, ncc);
        double c = mul(255.0, 1.0 < t ? 1.0 : t);
        c = c < 0.0 ? 0.0 : (255.0 < c ? 255.0 : c);
        return static_cast<int>(lround(c));
    }
}

template <int KIND, int WW, int WH>
__global__ void __launch_bounds__(kThreads) sweep_kernel(SweepArgs a) {
    using namespace dev;
    constexpr int RX = WW / 2, RY = WH / 2, NS = WW * WH;
    constexpr int NSP = KIND == FMVS_COST_NCC ? NS : 1;
    constexpr int kWarpsX = kThreads / 32;
    // per-warp segment state: every warp owns one 32-pixel row segment at a
    // time (no CTA barriers), so a level whose pixels are all narrow (the
    // tiled kernels own them) costs one coalesced metadata load and a vote
    // per segment
    __shared__ int s_prefix[kWarpsX][kSeg + 1];
    __shared__ int s_first[kWarpsX][kSeg];
    __shared__ uint32_t s_rel[kWarpsX][kSeg];
    __shared__ uint64_t s_bits[kWarpsX][kSeg];
    __shared__ double s_mean[kWarpsX][kSeg], s_var[kWarpsX][kSeg];
    __shared__ float s_patch[kWarpsX][kSeg][NSP];

    const int t = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const uint8_t* ref = a.ref_img;
    const int segs_per_row = (a.w + kSeg - 1) / kSeg;
    const int nseg = segs_per_row * a.h;
    for (int seg = blockIdx.x * kWarpsX + wp; seg < nseg; seg += gridDim.x * kWarpsX) {
        const int y = seg / segs_per_row;
        const int x0 = (seg - y * segs_per_row) * kSeg;
        const int npx = min(kSeg, a.w - x0);

        int cnt = 0;
        VolMeta m{0u, 0u};
        if (t < npx) {
            m = a.meta[static_cast<size_t>(y) * a.w + x0 + t];
            cnt = meta_count(m.fc);
            if (cnt <= a.exact_above)
                cnt = 0;  // narrow pixel: handled by the tiled certified kernel
        }
        if (!__any_sync(0xffffffffu, cnt > 0))
            continue;
        s_first[wp][t] = meta_first(m.fc);
        s_rel[wp][t] = m.rel;
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (t >= o)
                incl += v;
        }
        s_prefix[wp][t + 1] = incl;
        if (t == 0)
            s_prefix[wp][0] = 0;
        if (t < npx && cnt > 0) {
            const int x = x0 + t;
            if constexpr (KIND == FMVS_COST_CENSUS) {
                // census_bits_at (matching.cpp:28-42)
                const uint8_t c = ref[static_cast<size_t>(y) * a.w + x];
                uint64_t bits = 0;
                for (int dy = -RY; dy <= RY; ++dy)
                    for (int dx = -RX; dx <= RX; ++dx) {
                        if (dx == 0 && dy == 0)
                            continue;
                        const int xx = min(max(x + dx, 0), a.w - 1);
                        const int yy = min(max(y + dy, 0), a.h - 1);
                        bits = (bits << 1) | (ref[static_cast<size_t>(yy) * a.w + xx] < c ? 1u : 0u);
                    }
                s_bits[wp][t] = bits;
            } else {
                // reference patch, mean and two-pass variance (matching.cpp:199-210)
                int s = 0;
                for (int dy = -RY; dy <= RY; ++dy)
                    for (int dx = -RX; dx <= RX; ++dx) {
                        const int xx = min(max(x + dx, 0), a.w - 1);
                        const int yy = min(max(y + dy, 0), a.h - 1);
                        s_patch[wp][t][s++] = float(ref[static_cast<size_t>(yy) * a.w + xx]);
                    }
                double mean = 0.0, var = 0.0;
                for (int i = 0; i < NS; ++i)
                    mean = add(mean, double(s_patch[wp][t][i]));
                mean = div(mean, double(NS));
                for (int i = 0; i < NS; ++i) {
                    const double d = sub(double(s_patch[wp][t][i]), mean);
                    var = add(var, mul(d, d));
                }
                s_mean[wp][t] = mean;
                s_var[wp][t] = var;
            }
        }
        __syncwarp();

        const int total = s_prefix[wp][npx];
        const uint64_t base = a.row_base[y];
        for (int e = t; e < total; e += 32) {
            // pixel of entry e: largest j with prefix[j] <= e
            int lo = 0, hi = npx;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_prefix[wp][mid] <= e)
                    lo = mid;
                else
                    hi = mid;
            }
            const int j = lo;
            const int plane = s_first[wp][j] + (e - s_prefix[wp][j]);
            const double xd = double(x0 + j), yd = double(y);
            int sum_l = 0, sum_r = 0;
            for (int mm = 0; mm < a.nmatch; ++mm) {
                const int2 sz = a.sizes[mm];
                const int c = view_cost<KIND, WW, WH>(
                    a.quads[mm], sz.x, sz.y, a.homs + (static_cast<size_t>(mm) * a.nplanes + plane) * 9,
                    xd, yd, KIND == FMVS_COST_CENSUS ? s_bits[wp][j] : 0ull,
                    KIND == FMVS_COST_NCC ? s_patch[wp][j] : nullptr,
                    KIND == FMVS_COST_NCC ? s_mean[wp][j] : 0.0, KIND == FMVS_COST_NCC ? s_var[wp][j] : 0.0,
                    a.census_lut);
                if (mm < a.nleft)
                    sum_l += c;
                else
                    sum_r += c;
            }
            const uint64_t o = base + s_rel[wp][j] + (e - s_prefix[wp][j]);
            a.costs[o] = static_cast<uint16_t>(min(sum_l, sum_r));
        }
        __syncwarp();  // the segment's shared state is rewritten next iteration
    }
}

// ===================================================================
// Tiled certified census sweep (narrow pixels, count <= kNarrowMax).
//
// For a fixed (plane, view) the warped sample belonging to reference pixel
// (u, v) is the same bilinear lookup for every one of the WW*WH windows that
// contain (u, v); the reference recomputes it per window through its FP64
// walk. Here each CTA owns a 32x8 pixel tile, and for every plane of the
// union of its pixels' ranges it warps the (tile + halo) once per view in
// FP32 into shared memory, together with a rigorous bound E on
// |f32 - v64| valid for EVERY window's FP64 walk value (coordinate error from
// an anchored residual form of the homography, times the cell's bilinear
// Lipschitz constant, plus arithmetic slack). A census bit is taken from the
// FP32 values when |f_n - f_c| > E_n + E_c, which proves the FP64 comparison
// of the reference has the same outcome; otherwise that one bit is recomputed
// with the reference's exact FP64 walk. Costs are therefore bit-identical.
// ===================================================================

constexpr int kTW = 32, kTH = 8, kTiledThreads = kTW * kTH;
// resident CTAs per SM the census / NCC kernels are compiled for (register
// budget). Measured on B200 (C2): 3 CTAs (80 regs, few spills) 155 maps/s,
// 4 (64 regs) 164, 5 (48 regs, heavy spills) 165.6, 6 worse: latency hiding
// across the per-plane barriers beats spill traffic; with the exact-view
// path out of line, 4 and 5 tie (169-170) and 4 spills less. NCC box-sum
// kernel (c2ncc / C3): 2 CTAs 128.9 / 14.1, 3 137.6 / 15.8, 4 142.6 / 16.7
// (smem allows 4 for 5x5 windows).
#ifndef FMVS_CENSUS_MINB5
#define FMVS_CENSUS_MINB5 4
#endif
#ifndef FMVS_NCC_MINB
#define FMVS_NCC_MINB 4
#endif
#define FMVS_CENSUS_MINB(n) ((n) > 25 ? 2 : FMVS_CENSUS_MINB5)
// NCC 9x9 or > 4 matching views: shared memory admits only 2 / 3 CTAs per SM,
// so compiling them for 4 would only add spills
#define FMVS_NCC_MINB_OF(ns, nm) ((ns) > 25 ? 2 : ((nm) > 4 ? 3 : FMVS_NCC_MINB))
constexpr int kNarrowMax = 192;
constexpr int kMaxMatch = 8;

struct TileParams {
    float ax, bx, cx;  // r_x(du, dv) = q.x - xa * q.z
    float ay, by, cy;  // r_y(du, dv) = q.y - ya * q.z
    float az, bz, cz;  // q.z(du, dv)
    float dx, dy;      // certified coordinate error bounds (pixels)
    int xa, ya;        // integer anchors
    int exact;         // kTileExact: certification impossible, exact FP64 for this view;
                       // kTileInterior: the whole tile + halo warps strictly inside the view
};

constexpr int kTileExact = 1, kTileInterior = 2;

// kTileInterior test of a certified tile: a linear-fractional map with a
// positive denominator over a rectangle attains its coordinate extrema at the
// corners (its level sets are lines), so if the four corners land strictly
// inside [0, vw-1) x [0, vh-1) with the certified margins, no sample of the
// tile is clamped (pipeline bilinear, raster.hpp:71-84) and every window
// centre passes the reference's inside test (matching.cpp:224-231).
__device__ __forceinline__ bool tile_interior(const double* H, double U, double V, double DU, double DV,
                                              double dx, double dy, int vw, int vh) {
    double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const double uu = U + ((c & 1) ? DU : 0.0), vv = V + ((c & 2) ? DV : 0.0);
        const double qz = H[6] * uu + H[7] * vv + H[8];
        const double X = (H[0] * uu + H[1] * vv + H[2]) / qz;
        const double Y = (H[3] * uu + H[4] * vv + H[5]) / qz;
        xmin = fmin(xmin, X);
        xmax = fmax(xmax, X);
        ymin = fmin(ymin, Y);
        ymax = fmax(ymax, Y);
    }
    const double mx = dx + 1e-6, my = dy + 1e-6;  // + FP64 corner rounding (<< 1e-6)
    return xmin - mx > 0.0 && ymin - my > 0.0 && xmax + mx < double(vw - 1) &&
           ymax + my < double(vh - 1);
}

// FP64 sample of window position (i, j) of pixel (x, y), exactly as the
// reference computes it (matching.cpp:222-248).
__device__ __noinline__ double exact_window_sample(const double* __restrict__ hp,
                                                   const uint32_t* __restrict__ quad, int vw,
                                                   int vh, double xd, double yd, int rx, int ry,
                                                   int i, int j) {
    using namespace dev;
    double H[9];
    for (int k = 0; k < 9; ++k)
        H[k] = __ldg(hp + k);
    const double cx = add(add(mul(H[0], xd), mul(H[1], yd)), H[2]);
    const double cy = add(add(mul(H[3], xd), mul(H[4], yd)), H[5]);
    const double cz = add(add(mul(H[6], xd), mul(H[7], yd)), H[8]);
    double qx = sub(sub(cx, mul(double(rx), H[0])), mul(double(ry), H[1]));
    double qy = sub(sub(cy, mul(double(rx), H[3])), mul(double(ry), H[4]));
    double qz = sub(sub(cz, mul(double(rx), H[6])), mul(double(ry), H[7]));
    for (int r = 0; r < i; ++r) {
        qx = add(qx, H[1]);
        qy = add(qy, H[4]);
        qz = add(qz, H[7]);
    }
    for (int c = 0; c < j; ++c) {
        qx = add(qx, H[0]);
        qy = add(qy, H[3]);
        qz = add(qz, H[6]);
    }
    return warp_sample(quad, vw, vh, qx, qy, qz);
}

// The reference's inside test of the warped window centre (matching.cpp:224-231).
__device__ __noinline__ bool exact_inside(const double* __restrict__ hp, int vw, int vh, double xd,
                                          double yd) {
    using namespace dev;
    const double cx = add(add(mul(__ldg(hp + 0), xd), mul(__ldg(hp + 1), yd)), __ldg(hp + 2));
    const double cy = add(add(mul(__ldg(hp + 3), xd), mul(__ldg(hp + 4), yd)), __ldg(hp + 5));
    const double cz = add(add(mul(__ldg(hp + 6), xd), mul(__ldg(hp + 7), yd)), __ldg(hp + 8));
    if (!(cz > 0.0))
        return false;
    const double cxw = div(cx, cz), cyw = div(cy, cz);
    return cxw >= 0.0 && cyw >= 0.0 && cxw <= double(vw) - 1.0 && cyw <= double(vh) - 1.0;
}

// Byte k of q as a float, exactly (2^23 + b built by a byte permute, minus
// 2^23): two full-rate ALU/FMA instructions instead of a conversion.
template <int K>
__device__ __forceinline__ float byte_f(uint32_t q) {
    return __uint_as_float(__byte_perm(q, 0x4B000000u, 0x7540 | K)) - 8388608.0f;
}

// floor(t) for |t| < 2^22 without conversions: t + 1.5*2^23 rounded down has
// an ulp of 1, so its low mantissa bits are floor(t) (offset 0x4B400000).
__device__ __forceinline__ float floor_small(float t, int* it) {
    const float s = __fadd_rd(t, 12582912.0f);
    *it = __float_as_int(s) - 0x4B400000;
    return s - 12582912.0f;  // exact
}

// Same for doubles, |t| < 2^31: t + 1.5*2^52 rounded down, low word = floor(t).
__device__ __forceinline__ double floor_small(double t, int* it) {
    const double s = __dadd_rd(t, 6755399441055744.0);
    *it = __double2loint(s);
    return s - 6755399441055744.0;  // exact
}

// Per-(tile, plane, view) residual coefficients and error bounds (FP64).
__device__ TileParams make_tile_params(const double* __restrict__ hp, int u0, int v0, int du_max,
                                       int dv_max, int vw, int vh) {
    TileParams tp{};
    double H[9];
    for (int k = 0; k < 9; ++k)
        H[k] = __ldg(hp + k);
    const double U = u0, V = v0, DU = du_max, DV = dv_max;
    const double q0x = H[0] * U + H[1] * V + H[2];
    const double q0y = H[3] * U + H[4] * V + H[5];
    const double q0z = H[6] * U + H[7] * V + H[8];
    const double z10 = q0z + H[6] * DU, z01 = q0z + H[7] * DV, z11 = z10 + H[7] * DV;
    const double zmin = fmin(fmin(q0z, z10), fmin(z01, z11));
    const double two24 = 5.9604644775390625e-08;  // 2^-24
    const double two45 = 2.842170943040401e-14;   // 2^-45
    const double Mz = fabs(H[6]) * (fabs(U) + DU) + fabs(H[7]) * (fabs(V) + DV) + fabs(H[8]);
    const double Mx = fabs(H[0]) * (fabs(U) + DU) + fabs(H[1]) * (fabs(V) + DV) + fabs(H[2]);
    const double My = fabs(H[3]) * (fabs(U) + DU) + fabs(H[4]) * (fabs(V) + DV) + fabs(H[5]);
    if (!(zmin > 64.0 * two45 * Mz) || !(q0z > 0.0)) {
        tp.exact = 1;
        return tp;
    }
    double xa = floor(q0x / q0z), ya = floor(q0y / q0z);
    if (!(fabs(xa) < 4.0e6) || !(fabs(ya) < 4.0e6)) {
        tp.exact = 1;
        return tp;
    }
    const double axd = H[0] - xa * H[6], bxd = H[1] - xa * H[7], cxd = q0x - xa * q0z;
    const double ayd = H[3] - ya * H[6], byd = H[4] - ya * H[7], cyd = q0y - ya * q0z;
    const double Rx = fabs(axd) * DU + fabs(bxd) * DV + fabs(cxd);
    const double Ry = fabs(ayd) * DU + fabs(byd) * DV + fabs(cyd);
    const double Rz = fabs(H[6]) * DU + fabs(H[7]) * DV + fabs(q0z);
    // FP32 evaluation (coefficient rounding + two FMA roundings) and FP64
    // rounding of the coefficients / of the reference's own walk.
    const double ez = 4.0 * two24 * Rz + two45 * Mz;
    const double ex = 4.0 * two24 * Rx + two45 * (Mx + fabs(xa) * Mz);
    const double ey = 4.0 * two24 * Ry + two45 * (My + fabs(ya) * Mz);
    const double rzmin = zmin - ez;
    if (!(rzmin > 0.0)) {
        tp.exact = 1;
        return tp;
    }
    const double Tx = (Rx + ex) / rzmin, Ty = (Ry + ey) / rzmin;
    // division by rcp.approx (<= 2 ulp) + multiply (0.5 ulp): budget 8 ulp.
    double dx = (ex + Tx * ez) / rzmin + 8.0 * two24 * Tx +
                two45 * (Mx + (fabs(xa) + Tx) * Mz) / rzmin;
    double dy = (ey + Ty * ez) / rzmin + 8.0 * two24 * Ty +
                two45 * (My + (fabs(ya) + Ty) * Mz) / rzmin;
    dx = dx * 1.01 + 1e-9;
    dy = dy * 1.01 + 1e-9;
    if (!(dx < 0.05) || !(dy < 0.05)) {
        tp.exact = 1;
        return tp;
    }
    tp.ax = __double2float_rn(axd);
    tp.bx = __double2float_rn(bxd);
    tp.cx = __double2float_rn(cxd);
    tp.ay = __double2float_rn(ayd);
    tp.by = __double2float_rn(byd);
    tp.cy = __double2float_rn(cyd);
    tp.az = __double2float_rn(H[6]);
    tp.bz = __double2float_rn(H[7]);
    tp.cz = __double2float_rn(q0z);
    tp.dx = __double2float_ru(dx);
    tp.dy = __double2float_ru(dy);
    tp.xa = static_cast<int>(xa);
    tp.ya = static_cast<int>(ya);
    tp.exact = tile_interior(H, U, V, DU, DV, double(tp.dx), double(tp.dy), vw, vh) ? kTileInterior : 0;
    return tp;
}

// FP32 warp of tile sample (du, dv): cell-relative residual coordinates.
__device__ __forceinline__ void tile_coords(const TileParams& tp, float du, float dv, float* tx,
                                            float* ty) {
    const float rz = fmaf(tp.az, du, fmaf(tp.bz, dv, tp.cz));
    const float rx = fmaf(tp.ax, du, fmaf(tp.bx, dv, tp.cx));
    const float ry = fmaf(tp.ay, du, fmaf(tp.by, dv, tp.cy));
    const float r = __fdividef(1.0f, rz);
    *tx = rx * r;
    *ty = ry * r;
}

// Same as tile_coords with the reciprocal as one MUFU.RCP (rcp.approx.ftz:
// <= 1 ulp, inside the 8-ulp division budget of make_tile_params; rz is a
// normal positive float whenever the parameters are certified).
__device__ __forceinline__ void tile_coords_fast(const TileParams& tp, float du, float dv, float* tx,
                                                 float* ty) {
    const float rz = fmaf(tp.az, du, fmaf(tp.bz, dv, tp.cz));
    const float rx = fmaf(tp.ax, du, fmaf(tp.bx, dv, tp.cx));
    const float ry = fmaf(tp.ay, du, fmaf(tp.by, dv, tp.cy));
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(rz));
    *tx = rx * r;
    *ty = ry * r;
}

__device__ __forceinline__ int popcount_bits(uint32_t v) { return __popc(v); }
__device__ __forceinline__ int popcount_bits(uint64_t v) { return __popcll(v); }
__device__ __forceinline__ int lowest_bit(uint32_t v) { return __ffs(v) - 1; }
__device__ __forceinline__ int lowest_bit(uint64_t v) { return __ffsll(static_cast<long long>(v)) - 1; }

// Bit index of the census string (MSB = first window sample, centre skipped,
// matching.cpp:251-258) -> row-major window position.
template <int WW, int WH>
__device__ __forceinline__ int bit_to_pos(int bi) {
    constexpr int NB = WW * WH - 1, CENTER = (WW * WH) / 2;
    const int o = NB - 1 - bi;
    return o < CENTER ? o : o + 1;
}

constexpr int kItemCap = 1024;
constexpr int kPlaneChunk = 16;  // tile parameters computed for this many planes at once

// Dense levels (plane slicing): a CTA sweeps the same planes for all its
// pixels, one plane at a time, so direct u16 stores hit each pixel's run in a
// different sector per plane (C3: 3.3x the algorithmic DRAM bytes from
// partially written sectors evicted before completion). Each thread instead
// stages its pixel's costs of kRun consecutive planes in shared memory (its
// own row, stride chosen for conflict-free u16 stores) and writes them as one
// 32-byte run -- two 16-byte stores when the run is full and aligned.
// Census kernels stage 16 planes (32-byte runs); the NCC kernel 8 (16-byte
// runs: its shared memory would otherwise drop it from 4 to 3 CTAs per SM).
// Row stride kRun + 2 u16: an odd number of words, so the u16 stores of a
// warp's 32 threads hit distinct banks.
constexpr int kRun = 16, kRunNcc = 8;

// Writes the staged costs of planes [c0, p] that lie in the pixel's range.
template <int RUN>
__device__ __forceinline__ void flush_run(uint16_t* __restrict__ costs, const uint16_t* run, int c0, int p,
                                          int first, int count, uint64_t base) {
    const int lo = max(c0, first), hi = min(p, first + count - 1);
    if (lo > hi)
        return;
    const uint64_t o = base + static_cast<uint64_t>(lo - first);
    if (hi - lo + 1 == RUN && (o & 7) == 0) {
        const uint32_t* r = reinterpret_cast<const uint32_t*>(run);  // lo == c0: the whole row
        uint4* dst = reinterpret_cast<uint4*>(costs + o);
#pragma unroll
        for (int q = 0; q < RUN / 8; ++q)
            dst[q] = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
    } else {
        for (int q = lo; q <= hi; ++q)
            costs[base + static_cast<uint64_t>(q - first)] = run[q - c0];
    }
}

struct ViewConst {
    const uint32_t* quad;
    const double* homs;  // homs of this view, plane 0
    int w, h;
    int left;            // 1 if the view lies left of the reference
};

// FP64-coordinate variant of the tile parameters: the residual form is
// evaluated in FP64 (3 FMA + a correctly rounded reciprocal), so the certified
// coordinate error is ~1e-10 px and a sample's value bound collapses to the
// FP32 bilinear arithmetic (~4e-5). Used by the NCC kernel, whose cost is a
// smooth function of all samples and needs tight per-sample bounds.
struct TileParams64 {
    double ax, bx, cx, ay, by, cy, az, bz, cz;
    float dx, dy;
    float eb;  // tile-uniform sample bound, or < 0: per-sample bounds
    int xa, ya;
    int exact;
};

__device__ TileParams64 make_tile_params64(const double* __restrict__ hp, int u0, int v0,
                                           int du_max, int dv_max, int vw, int vh) {
    TileParams64 tp{};
    double H[9];
    for (int k = 0; k < 9; ++k)
        H[k] = __ldg(hp + k);
    const double U = u0, V = v0, DU = du_max, DV = dv_max;
    const double q0x = H[0] * U + H[1] * V + H[2];
    const double q0y = H[3] * U + H[4] * V + H[5];
    const double q0z = H[6] * U + H[7] * V + H[8];
    const double z10 = q0z + H[6] * DU, z01 = q0z + H[7] * DV, z11 = z10 + H[7] * DV;
    const double zmin = fmin(fmin(q0z, z10), fmin(z01, z11));
    const double two45 = 2.842170943040401e-14;   // 2^-45
    const double two49 = 1.7763568394002505e-15;  // 2^-49
    const double Mz = fabs(H[6]) * (fabs(U) + DU) + fabs(H[7]) * (fabs(V) + DV) + fabs(H[8]);
    const double Mx = fabs(H[0]) * (fabs(U) + DU) + fabs(H[1]) * (fabs(V) + DV) + fabs(H[2]);
    const double My = fabs(H[3]) * (fabs(U) + DU) + fabs(H[4]) * (fabs(V) + DV) + fabs(H[5]);
    if (!(zmin > 64.0 * two45 * Mz) || !(q0z > 0.0)) {
        tp.exact = 1;
        return tp;
    }
    const double xa = floor(q0x / q0z), ya = floor(q0y / q0z);
    if (!(fabs(xa) < 4.0e6) || !(fabs(ya) < 4.0e6)) {
        tp.exact = 1;
        return tp;
    }
    tp.ax = H[0] - xa * H[6];
    tp.bx = H[1] - xa * H[7];
    tp.cx = q0x - xa * q0z;
    tp.ay = H[3] - ya * H[6];
    tp.by = H[4] - ya * H[7];
    tp.cy = q0y - ya * q0z;
    tp.az = H[6];
    tp.bz = H[7];
    tp.cz = q0z;
    const double Rx = fabs(tp.ax) * DU + fabs(tp.bx) * DV + fabs(tp.cx);
    const double Ry = fabs(tp.ay) * DU + fabs(tp.by) * DV + fabs(tp.cy);
    const double Rz = fabs(H[6]) * DU + fabs(H[7]) * DV + fabs(q0z);
    // FP64 coefficient construction + FMA evaluation (generous 16 ulp) and the
    // reference's own FP64 walk rounding (2^-45 relative to the magnitudes)
    const double ez = two49 * (Rz + Mz) + two45 * Mz;
    const double ex = two49 * (Rx + Mx + fabs(xa) * Mz) + two45 * (Mx + fabs(xa) * Mz);
    const double ey = two49 * (Ry + My + fabs(ya) * Mz) + two45 * (My + fabs(ya) * Mz);
    const double rzmin = zmin - ez;
    if (!(rzmin > 0.0)) {
        tp.exact = 1;
        return tp;
    }
    const double Tx = (Rx + ex) / rzmin, Ty = (Ry + ey) / rzmin;
    // reciprocal (Newton, < 2^-47) and product rounding of tile_coords64
    const double two46 = 1.4210854715202004e-14;  // 2^-46
    double dx = (ex + Tx * ez) / rzmin + two46 * Tx + 1e-12;
    double dy = (ey + Ty * ez) / rzmin + two46 * Ty + 1e-12;
    dx *= 1.01;
    dy *= 1.01;
    if (!(dx < 1e-3) || !(dy < 1e-3)) {
        tp.exact = 1;
        return tp;
    }
    tp.dx = __double2float_ru(dx);
    tp.dy = __double2float_ru(dy);
    // The bilinear interpolant of byte images is 255-Lipschitz along each
    // axis, across cell edges and clamped borders included, so 255*(dx + dy)
    // bounds the effect of the coordinate error on every sample of the tile;
    // + the float cast of the cell fraction (<= 2^-25 per axis) and the FP32
    // bilinear arithmetic (< 4e-5, see ncc_sample). When the coordinate term
    // is negligible (the usual ~1e-10 px) this tile-wide bound replaces the
    // per-sample ones.
    const float lip = 255.0f * (tp.dx + tp.dy);
    tp.eb = lip < 1.0e-5f ? (lip + 255.0f * 6.0e-8f + 4.0e-5f) * 1.0001f : -1.0f;
    tp.xa = static_cast<int>(xa);
    tp.ya = static_cast<int>(ya);
    tp.exact = tile_interior(H, U, V, DU, DV, double(tp.dx), double(tp.dy), vw, vh) ? kTileInterior : 0;
    return tp;
}

__device__ __forceinline__ void tile_coords64(const TileParams64& tp, double du, double dv,
                                              double* tx, double* ty) {
    const double rz = fma(tp.az, du, fma(tp.bz, dv, tp.cz));
    const double rx = fma(tp.ax, du, fma(tp.bx, dv, tp.cx));
    const double ry = fma(tp.ay, du, fma(tp.by, dv, tp.cy));
    // 1/rz: MUFU seed + two Newton steps (relative error < 2^-47 for any
    // seed error < 2^-12; budgeted in make_tile_params64) instead of the
    // correctly rounded reciprocal's longer sequence
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(rz));
    r = fma(r, fma(-rz, r, 1.0), r);
    r = fma(r, fma(-rz, r, 1.0), r);
    *tx = rx * r;
    *ty = ry * r;
}

// (value, bound) of one FP64-coordinate tile sample: FP32 bilinear of the
// cell quad q at (ax, ay); the bound is the cell's Lipschitz constant times
// the coordinate error (255 within the error of a cell edge) plus the FP32
// bilinear rounding.
// BOUND false: the value only (tiles with a uniform bound, TileParams64::eb).
template <bool BOUND>
__device__ __forceinline__ float2 ncc_sample(uint32_t q, float ax, float ay, float dx, float dy) {
    const float i00 = byte_f<0>(q), i10 = byte_f<1>(q), i01 = byte_f<2>(q), i11 = byte_f<3>(q);
    const float top = fmaf(ax, i10 - i00, i00);
    const float bot = fmaf(ax, i11 - i01, i01);
    const float f = fmaf(ay, bot - top, top);
    if (!BOUND)
        return make_float2(f, 0.0f);
    // the float cast of (t - floor t) adds 2^-24 to the coordinate error; a
    // negative dx / dy marks an axis certainly clamped at the view edge (the
    // sample does not depend on it: no error along it)
    const float ddx = dx < 0.0f ? 0.0f : dx + 6.0e-8f, ddy = dy < 0.0f ? 0.0f : dy + 6.0e-8f;
    const bool near_x = ax < ddx || ax > 1.0f - ddx;
    const bool near_y = ay < ddy || ay > 1.0f - ddy;
    const float gx = near_x ? 255.0f : fmaxf(fabsf(i10 - i00), fabsf(i11 - i01));
    const float gy = near_y ? 255.0f : fmaxf(fabsf(i01 - i00), fabsf(i11 - i10));
    // FP32 bilinear: 3 FMA + 2 SUB roundings on values <= 255 (< 4e-5)
    return make_float2(f, fmaf(gx, ddx, fmaf(gy, ddy, 4.0e-5f)));
}

// Sample of the tile at (du, dv): FP64 residual coordinates, FP32 bilinear;
// returns (value, bound) like the FP32-coordinate path.
template <bool BOUND>
__device__ __forceinline__ float2 tile_sample64(const TileParams64& tp, const ViewConst& vc,
                                                double du, double dv, uint8_t* in_flag) {
    double tx, ty;
    tile_coords64(tp, du, dv, &tx, &ty);
    {
        // certified inside test of this sample as a window centre
        // (matching.cpp:224-231): 1 inside, 0 outside, 2 undecided
        const double X = double(tp.xa) + tx, Y = double(tp.ya) + ty;
        const double ddx = double(tp.dx) + 1e-9, ddy = double(tp.dy) + 1e-9;
        const double wm = double(vc.w - 1), hm = double(vc.h - 1);
        uint8_t fl = 2;
        if (X - ddx >= 0.0 && Y - ddy >= 0.0 && X + ddx <= wm && Y + ddy <= hm)
            fl = 1;
        else if (X + ddx < 0.0 || Y + ddy < 0.0 || X - ddx > wm || Y - ddy > hm)
            fl = 0;
        *in_flag = fl;
    }
    const double fx = floor(tx), fy = floor(ty);
    int X0 = tp.xa + static_cast<int>(fx), Y0 = tp.ya + static_cast<int>(fy);
    float ax = __double2float_rn(tx - fx), ay = __double2float_rn(ty - fy);
    // edge clamp (raster.hpp:71-84); a coordinate certainly past the edge
    // leaves the reference's sample independent of it (see the census path)
    float ddx = tp.dx, ddy = tp.dy;
    const double ex = double(tp.dx) + 1e-9, ey = double(tp.dy) + 1e-9;
    if (X0 < 0) {
        X0 = 0;
        ax = 0.0f;
        if (double(tp.xa) + tx + ex < 0.0)
            ddx = -1.0f;
    } else if (X0 >= vc.w - 1) {
        X0 = vc.w - 1;
        ax = 0.0f;
        if (double(tp.xa) + tx - ex >= double(vc.w - 1))
            ddx = -1.0f;
    }
    if (Y0 < 0) {
        Y0 = 0;
        ay = 0.0f;
        if (double(tp.ya) + ty + ey < 0.0)
            ddy = -1.0f;
    } else if (Y0 >= vc.h - 1) {
        Y0 = vc.h - 1;
        ay = 0.0f;
        if (double(tp.ya) + ty - ey >= double(vc.h - 1))
            ddy = -1.0f;
    }
    return ncc_sample<BOUND>(__ldg(vc.quad + static_cast<uint32_t>(Y0 * vc.w + X0)), ax, ay, ddx, ddy);
}

// tile_sample64 of a kTileInterior tile: no clamping, no inside flag.
template <bool BOUND>
__device__ __forceinline__ float2 tile_sample64_interior(const TileParams64& tp, const ViewConst& vc,
                                                         double du, double dv) {
    double tx, ty;
    tile_coords64(tp, du, dv, &tx, &ty);
    int ix, iy;  // |tx|, |ty| < view size (interior tile)
    const double fx = floor_small(tx, &ix), fy = floor_small(ty, &iy);
    const int X0 = tp.xa + ix, Y0 = tp.ya + iy;
    const float ax = __double2float_rn(tx - fx), ay = __double2float_rn(ty - fy);
    return ncc_sample<BOUND>(__ldg(vc.quad + static_cast<uint32_t>(Y0 * vc.w + X0)), ax, ay, tp.dx, tp.dy);
}

// One view's part of the NCC tile build (this thread's samples r, r + KTPV,
// ...): quantised samples F = rint(f * 2^16) into t, inside flags into fl
// (general tiles); returns the thread's max sample bound.
template <bool BOUND, int SW, int SN, int KTPV>
__device__ __forceinline__ float build_ncc_tile(const TileParams64& tp, const ViewConst& vc, int* t,
                                                uint8_t* fl, int r) {
    int dv = r / SW, du = r - dv * SW;
    float emax = BOUND ? 0.0f : tp.eb;
    for (; r < SN; r += KTPV) {
        float2 v;
        if (tp.exact == kTileInterior) {
            v = tile_sample64_interior<BOUND>(tp, vc, double(du), double(dv));
        } else {
            uint8_t f = 2;
            v = tile_sample64<BOUND>(tp, vc, double(du), double(dv), &f);
            fl[r] = f;
        }
        t[r] = __float2int_rn(v.x * 65536.0f);  // exact scaling, |F/2^16 - f| <= 2^-17
        if (BOUND)
            emax = fmaxf(emax, v.y);
        du += KTPV % SW;
        dv += KTPV / SW;
        if (du >= SW) {
            du -= SW;
            ++dv;
        }
    }
    return emax;
}

// Exact FP64 census cost of one view (views whose tile certification is
// impossible; rare). Out of line so its registers do not weigh on the tiled
// kernel's hot loop.
template <int WW, int WH>
__device__ __noinline__ int census_view_exact(const uint32_t* __restrict__ quad, int vw, int vh,
                                              const double* __restrict__ hp, double xd, double yd,
                                              uint64_t ref_bits, const uint16_t* __restrict__ lut) {
    return view_cost<FMVS_COST_CENSUS, WW, WH>(quad, vw, vh, hp, xd, yd, ref_bits, nullptr, 0.0, 0.0,
                                               lut);
}

// Interval [lo, hi] of every FP64 walk value of one tile sample (outward
// rounded): FP32 bilinear of the cell quad q at (ax, ay) widened by the cell's
// Lipschitz constant times the certified coordinate error (255 when the
// sample is within the error of a cell edge).
__device__ __forceinline__ float2 census_sample(uint32_t q, float ax, float ay, float dx, float dy) {
    const float i00 = byte_f<0>(q), i10 = byte_f<1>(q), i01 = byte_f<2>(q), i11 = byte_f<3>(q);
    const float top = fmaf(ax, i10 - i00, i00);
    const float bot = fmaf(ax, i11 - i01, i01);
    const float f = fmaf(ay, bot - top, top);
    const bool near_x = ax < dx || ax > 1.0f - dx;
    const bool near_y = ay < dy || ay > 1.0f - dy;
    const float gx = near_x ? 255.0f : fmaxf(fabsf(i10 - i00), fabsf(i11 - i01));
    const float gy = near_y ? 255.0f : fmaxf(fabsf(i01 - i00), fabsf(i11 - i10));
    // FP32 bilinear rounding: the tap differences are exact, top / bot / f
    // each round once (<= 2^-17 below 256) and bot - top once, carrying the
    // errors of top and bot: |f - f_exact| <= 5 * 2^-17 < 4e-5 (the
    // reference's FP64 bilinear adds < 1e-13). No zero bound even for a flat
    // cell: the reference's (1 - a) * I + a * I is not always exactly I in
    // FP64 (a with bits below 2^-52, i.e. coordinates below 1).
    const float e = fmaf(gx, dx, fmaf(gy, dy, 4.0e-5f));
    return make_float2(__fsub_rd(f, e), __fadd_ru(f, e));
}

template <int WW, int WH, int NM>
__global__ void __launch_bounds__(kTiledThreads, FMVS_CENSUS_MINB(WW * WH)) sweep_census_tiled(SweepArgs a) {
    using namespace dev;
    using BitsT = typename std::conditional<(WW * WH - 1 > 32), uint64_t, uint32_t>::type;
    constexpr int RX = WW / 2, RY = WH / 2;
    constexpr int SW = kTW + WW - 1, SH = kTH + WH - 1, SN = SW * SH;
    constexpr int CENTER = (WW * WH) / 2;
    extern __shared__ float2 s_tile[];  // [NM][SH][SW] (value, bound) of the warped tile + halo
    __shared__ TileParams s_tp[kPlaneChunk][NM];
    __shared__ ViewConst s_vc[NM];
    __shared__ uint8_t s_inflag[NM * kTW * kTH];  // certified inside flag of each window centre
    constexpr int kTPV = kTiledThreads / NM;      // tile-build threads per view
    __shared__ int s_pmin, s_pmax;
    __shared__ int s_count;  // exact samples listed for the current plane
    __shared__ uint32_t s_items[kItemCap];  // (thread, view, window position)
    __shared__ double s_vals[kItemCap];     // their exact FP64 samples
    __shared__ uint16_t s_lut[WW * WH];     // census cost LUT (popcount -> cost)
    __shared__ __align__(16) uint16_t s_run[kTiledThreads * (kRun + 2)];  // dense levels: staged runs

    const int tx = threadIdx.x % kTW, ty = threadIdx.x / kTW;
    const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH;
    const int x = x0 + tx, y = y0 + ty;
    const bool in_img = x < a.w && y < a.h;

    int first = 0, count = 0;
    uint64_t base = 0;
    BitsT ref_bits = 0;
    if (in_img) {
        const VolMeta m = a.meta[static_cast<size_t>(y) * a.w + x];
        first = meta_first(m.fc);
        count = meta_count(m.fc);
        base = a.row_base[y] + m.rel;
        if (count > a.exact_above)
            count = 0;  // wide pixel: the exact per-hypothesis kernel owns it
        if (count > 0) {
            const uint8_t* ref = a.ref_img;  // census_bits_at (matching.cpp:28-42)
            const uint8_t c = ref[static_cast<size_t>(y) * a.w + x];
            for (int dy = -RY; dy <= RY; ++dy)
                for (int dx = -RX; dx <= RX; ++dx) {
                    if (dx == 0 && dy == 0)
                        continue;
                    const int xx = min(max(x + dx, 0), a.w - 1);
                    const int yy = min(max(y + dy, 0), a.h - 1);
                    ref_bits = (ref_bits << 1) | (ref[static_cast<size_t>(yy) * a.w + xx] < c ? 1u : 0u);
                }
        }
    }
    if (threadIdx.x == 0) {
        s_pmin = 0x7FFFFFFF;
        s_pmax = -1;
        s_count = 0;
    }
    if (threadIdx.x < NM) {
        const int m = threadIdx.x;
        const int2 sz = a.sizes[m];
        s_vc[m] = ViewConst{a.quads[m], a.homs + static_cast<size_t>(m) * a.nplanes * 9, sz.x, sz.y,
                            m < a.nleft ? 1 : 0};
    }
    if (threadIdx.x < WW * WH)
        s_lut[threadIdx.x] = a.census_lut[threadIdx.x];  // entries 0 .. WW*WH-1 (popcounts)
    __syncthreads();
    if (count > 0) {
        atomicMin(&s_pmin, first);
        atomicMax(&s_pmax, first + count - 1);
    }
    __syncthreads();
    // plane slice of this CTA (gridDim.z > 1 splits dense levels across CTAs)
    const int slice = (a.nplanes + gridDim.z - 1) / gridDim.z;
    const int pmin = max(s_pmin, static_cast<int>(blockIdx.z) * slice);
    const int pmax = min(s_pmax, static_cast<int>(blockIdx.z + 1) * slice - 1);
    const double xd = double(x), yd = double(y);

    for (int p = pmin; p <= pmax; ++p) {
        const bool need = count > 0 && p >= first && p < first + count;
        const int slot = (p - pmin) % kPlaneChunk;
        if (slot == 0) {
            // tile parameters of the next kPlaneChunk planes x NM views, in
            // parallel (the previous chunk's were last read in pass 1 of the
            // previous plane, before its barrier I)
            for (int k = threadIdx.x; k < kPlaneChunk * NM; k += kTiledThreads) {
                const int pp = p + k / NM, m = k % NM;
                if (pp <= pmax)
                    s_tp[k / NM][m] = make_tile_params(s_vc[m].homs + static_cast<size_t>(pp) * 9,
                                                       x0 - RX, y0 - RY, SW - 1, SH - 1, s_vc[m].w,
                                                       s_vc[m].h);
            }
            __syncthreads();
        }
        // Three barriers per plane: tile complete (T), exact-sample list
        // complete (I), exact samples taken (P). The tile of plane p+1 may be
        // built while slower warps finish pass 3 of plane p: pass 3 reads
        // neither the tile nor the inside flags, and every warp finished
        // reading them (pass 1) before barrier I of plane p.
        if (a.stats && threadIdx.x == 0)
            atomicAdd(a.stats + 4, 1ull);
        // ---- warp the tile + halo of every matching view into shared memory.
        // Each thread serves one view (its tile parameters stay in registers)
        // and strides over that view's samples; interior samples also record
        // the certified inside flag of the window centre (matching.cpp:224-231).
        if (threadIdx.x < NM * kTPV) {
            const int m = threadIdx.x / kTPV;
            const TileParams tp = s_tp[slot][m];
            float2* t = s_tile + m * SN;
            uint8_t* fl = s_inflag + m * (kTW * kTH);
            if (tp.exact == kTileExact) {
                for (int r = threadIdx.x - m * kTPV; r < SN; r += kTPV)
                    t[r] = make_float2(0.0f, 1e30f);
            } else if (tp.exact == kTileInterior) {
                // no clamping, no inside flags (tile_interior)
                const uint32_t* quad = s_vc[m].quad;
                const int vw = s_vc[m].w;
                int r = threadIdx.x - m * kTPV;
                int dv = r / SW, du = r - dv * SW;
                for (; r < SN; r += kTPV) {
                    float tcx, tcy;
                    tile_coords_fast(tp, float(du), float(dv), &tcx, &tcy);
                    int ix, iy;  // |tcx|, |tcy| < view size (interior tile)
                    const float fx = floor_small(tcx, &ix), fy = floor_small(tcy, &iy);
                    const int X0 = tp.xa + ix, Y0 = tp.ya + iy;
                    const float ax = tcx - fx, ay = tcy - fy;
                    t[r] = census_sample(__ldg(quad + (Y0 * vw + X0)), ax, ay, tp.dx, tp.dy);
                    du += kTPV % SW;
                    dv += kTPV / SW;
                    if (du >= SW) {
                        du -= SW;
                        ++dv;
                    }
                }
            } else {
                const uint32_t* quad = s_vc[m].quad;
                const int vw = s_vc[m].w, vh = s_vc[m].h;
                const float xlo = float(-tp.xa), xhi = float(vw - 1 - tp.xa);
                const float ylo = float(-tp.ya), yhi = float(vh - 1 - tp.ya);
                int r = threadIdx.x - m * kTPV;
                int dv = r / SW, du = r - dv * SW;
                for (; r < SN; r += kTPV) {
                    float tcx, tcy;
                    tile_coords_fast(tp, float(du), float(dv), &tcx, &tcy);
                    if (du >= RX && du < RX + kTW && dv >= RY && dv < RY + kTH) {
                        uint8_t f = 2;  // undecided -> exact test in pass 1
                        if (tcx - tp.dx >= xlo && tcy - tp.dy >= ylo && tcx + tp.dx <= xhi &&
                            tcy + tp.dy <= yhi)
                            f = 1;  // (float ops above are exact or err toward ambiguity)
                        else if (tcx + tp.dx < xlo || tcy + tp.dy < ylo || tcx - tp.dx > xhi ||
                                 tcy - tp.dy > yhi)
                            f = 0;
                        fl[(dv - RY) * kTW + du - RX] = f;
                    }
                    const float fx = floorf(tcx), fy = floorf(tcy);
                    int X0 = tp.xa + static_cast<int>(fx), Y0 = tp.ya + static_cast<int>(fy);
                    float ax = tcx - fx, ay = tcy - fy;
                    // edge clamp (raster.hpp:71-84). When the reference's
                    // coordinate is CERTAINLY past the edge its sample does not
                    // depend on that coordinate at all (a = 0 there too): no
                    // coordinate error along that axis (otherwise the clamped
                    // a = 0 reads as "near a cell edge", Lipschitz 255)
                    float ddx = tp.dx, ddy = tp.dy;
                    if (X0 < 0) {
                        X0 = 0;
                        ax = 0.0f;
                        if (__fadd_ru(tcx, tp.dx) < xlo)
                            ddx = 0.0f;
                    } else if (X0 >= vw - 1) {
                        X0 = vw - 1;
                        ax = 0.0f;
                        if (__fsub_rd(tcx, tp.dx) >= xhi)
                            ddx = 0.0f;
                    }
                    if (Y0 < 0) {
                        Y0 = 0;
                        ay = 0.0f;
                        if (__fadd_ru(tcy, tp.dy) < ylo)
                            ddy = 0.0f;
                    } else if (Y0 >= vh - 1) {
                        Y0 = vh - 1;
                        ay = 0.0f;
                        if (__fsub_rd(tcy, tp.dy) >= yhi)
                            ddy = 0.0f;
                    }
                    t[r] = census_sample(__ldg(quad + (Y0 * vw + X0)), ax, ay, ddx, ddy);
                    du += kTPV % SW;
                    dv += kTPV / SW;
                    if (du >= SW) {
                        du -= SW;
                        ++dv;
                    }
                }
            }
        }
        __syncthreads();  // T
        if (a.stats && need)
            atomicAdd(a.stats + 7, 1ull);  // useful (pixel, plane) slots of the iteration
        // ---- pass 1: FP32 census bits; undecided-bit masks only where needed
        BitsT bits[NM], uns[NM];
        uint32_t view_out = 0;    // bit m: window centre outside the view -> 255
        uint32_t view_exact = 0;  // bit m: certification impossible -> exact path
        int my_items = 0;
#pragma unroll
        for (int m = 0; m < NM; ++m) {
            bits[m] = 0;
            uns[m] = 0;
            if (!need)
                continue;
            const int tpe = s_tp[slot][m].exact;
            if (tpe == kTileExact) {
                view_exact |= 1u << m;
                continue;
            }
            const ViewConst& vc = s_vc[m];
            // inside test of the window centre (matching.cpp:224-231), certified
            // in the tile build; undecided -> the reference's exact FP64 test
            bool inside = true;
            if (tpe != kTileInterior) {
                const uint8_t fl = s_inflag[m * (kTW * kTH) + threadIdx.x];
                inside = fl == 2 ? exact_inside(vc.homs + static_cast<size_t>(p) * 9, vc.w, vc.h, xd, yd)
                                 : fl == 1;
            }
            if (!inside) {
                view_out |= 1u << m;
                continue;
            }
            const float2* t = s_tile + m * SN;
            const float2 c = t[(ty + RY) * SW + tx + RX];  // (lo, hi) of the centre
            BitsT lt = 0, nge = 0;
#pragma unroll
            for (int i = 0; i < WH; ++i)
#pragma unroll
                for (int j = 0; j < WW; ++j) {
                    if (i * WW + j == CENTER)
                        continue;
                    const float2 n = t[(ty + i) * SW + tx + j];
                    // certified n < c  <=>  hi_n < lo_c  <=>  sign(hi_n - lo_c);
                    // certified n >= c <=>  lo_n >= hi_c <=> !sign(lo_n - hi_c)
                    // (float subtraction is exactly sign-correct; lo, hi > -0
                    // except lo = -0, which only makes the test more cautious)
                    lt = (lt << 1) | static_cast<BitsT>(__float_as_uint(n.y - c.x) >> 31);
                    nge = (nge << 1) | static_cast<BitsT>(__float_as_uint(n.x - c.y) >> 31);
                }
            constexpr BitsT kAll = static_cast<BitsT>(~BitsT(0)) >> (sizeof(BitsT) * 8 - (WW * WH - 1));
            const BitsT u = ~lt & nge & kAll;
            bits[m] = lt;
            uns[m] = u;
            if (u)
                my_items += 1 + popcount_bits(u);
            if (a.stats) {
                atomicAdd(a.stats + 0, 1ull);
                if (uns[m]) {
                    atomicAdd(a.stats + 1, 1ull);
                    atomicAdd(a.stats + 2, static_cast<unsigned long long>(popcount_bits(uns[m])));
                }
            }
        }
        // ---- pass 1a: only undecided views that can change min(sum_l, sum_r)
        // need resolving. A view's cost lies in [lut[h_sure], lut[h_sure +
        // #undecided]] (the census LUT is monotone); a side whose lower bound
        // reaches the other side's upper bound is never the strict minimum's
        // only source, so its undecided bits may take any completion (the
        // FP32 guess) without changing the u16 cost.
        if (my_items && !a.plane_slicing) {  // refined levels (measured: no gain on dense ones)
            int lo_l = 0, hi_l = 0, lo_r = 0, hi_r = 0;
#pragma unroll
            for (int m = 0; m < NM; ++m) {
                int lo, hi;
                if ((view_exact >> m) & 1u) {
                    lo = 0;
                    hi = 255;
                } else if ((view_out >> m) & 1u) {
                    lo = hi = 255;
                } else {
                    const int hs = popcount_bits((bits[m] ^ ref_bits) & ~uns[m]);
                    lo = s_lut[hs];
                    hi = s_lut[hs + popcount_bits(uns[m])];
                }
                if (m < a.nleft) {  // views 0..nleft-1 lie left of the reference
                    lo_l += lo;
                    hi_l += hi;
                } else {
                    lo_r += lo;
                    hi_r += hi;
                }
            }
            const bool rel_l = lo_l < hi_r, rel_r = lo_r < hi_l;
            my_items = 0;
#pragma unroll
            for (int m = 0; m < NM; ++m) {
                if (!(m < a.nleft ? rel_l : rel_r))
                    uns[m] = 0;
                if (uns[m])
                    my_items += 1 + popcount_bits(uns[m]);
            }
        }
        // ---- pass 1b: CTA-wide list of the samples that need the exact walk
        // (slots allocated with a shared-memory atomic: the list order varies,
        // each thread reads back exactly its own slots)
        int off = 0;
        if (my_items)
            off = atomicAdd(&s_count, my_items);
        if (my_items) {
            int k = off;
#pragma unroll
            for (int m = 0; m < NM; ++m) {
                if (!uns[m])
                    continue;
                if (k < kItemCap)
                    s_items[k] = threadIdx.x | (m << 8) | (CENTER << 12);
                ++k;
                BitsT u = uns[m];
                while (u) {
                    const int bi = lowest_bit(u);
                    u &= u - 1;
                    if (k < kItemCap)
                        s_items[k] = threadIdx.x | (m << 8) | (bit_to_pos<WW, WH>(bi) << 12);
                    ++k;
                }
            }
        }
        __syncthreads();  // I
        // ---- pass 2: exact FP64 samples, one per thread (fully SIMT-parallel)
        const int total = s_count;
        const int nitems = min(total, kItemCap);
        if (a.stats && threadIdx.x == 0)
            atomicAdd(a.stats + 6, static_cast<unsigned long long>(total));
        for (int it = threadIdx.x; it < nitems; it += kTiledThreads) {
            const uint32_t item = s_items[it];
            const int t = item & 0xFF, m = (item >> 8) & 0xF, pos = item >> 12;
            const ViewConst& vc = s_vc[m];
            s_vals[it] = exact_window_sample(vc.homs + static_cast<size_t>(p) * 9, vc.quad, vc.w,
                                             vc.h, double(x0 + t % kTW), double(y0 + t / kTW), RX,
                                             RY, pos / WW, pos % WW);
        }
        __syncthreads();  // P
        if (threadIdx.x == 0)
            s_count = 0;  // next plane allocates after its barrier T
        // ---- pass 3: resolve undecided bits, per-side sums, min -> u16
        if (need) {
            int sum_l = 0, sum_r = 0, k = off;
#pragma unroll
            for (int m = 0; m < NM; ++m) {
                const ViewConst& vc = s_vc[m];
                int cost;
                if ((view_exact >> m) & 1u) {
                    if (a.stats)
                        atomicAdd(a.stats + 3, 1ull);
                    cost = census_view_exact<WW, WH>(vc.quad, vc.w, vc.h,
                                                     vc.homs + static_cast<size_t>(p) * 9, xd, yd,
                                                     ref_bits, a.census_lut);
                } else if ((view_out >> m) & 1u) {
                    cost = 255;
                } else {
                    BitsT b = bits[m];
                    if (uns[m]) {
                        const double* hp = vc.homs + static_cast<size_t>(p) * 9;
                        const double wc = k < kItemCap ? s_vals[k]
                                                       : exact_window_sample(hp, vc.quad, vc.w, vc.h,
                                                                             xd, yd, RX, RY, RY, RX);
                        ++k;
                        BitsT u = uns[m];
                        while (u) {
                            const int bi = lowest_bit(u);
                            u &= u - 1;
                            const int pos = bit_to_pos<WW, WH>(bi);
                            const double v = k < kItemCap
                                                 ? s_vals[k]
                                                 : exact_window_sample(hp, vc.quad, vc.w, vc.h, xd, yd,
                                                                       RX, RY, pos / WW, pos % WW);
                            ++k;
                            const BitsT one = 1;
                            b = v < wc ? (b | (one << bi)) : (b & ~(one << bi));
                        }
                    }
                    cost = s_lut[popcount_bits(b ^ ref_bits)];
                }
                if (m < a.nleft)
                    sum_l += cost;
                else
                    sum_r += cost;
            }
            const uint16_t v = static_cast<uint16_t>(min(sum_l, sum_r));
            if (a.plane_slicing)
                s_run[threadIdx.x * (kRun + 2) + (p - pmin) % kRun] = v;
            else
                a.costs[base + static_cast<uint64_t>(p - first)] = v;
        }
        if (a.plane_slicing && ((p - pmin) % kRun == kRun - 1 || p == pmax))
            flush_run<kRun>(a.costs, s_run + threadIdx.x * (kRun + 2), p - (p - pmin) % kRun, p, first, count,
                            base);
    }
}

// ===================================================================
// Tiled certified NCC sweep. Same tile warp as the census kernel (FP64 tile
// coordinates). Each tile sample is quantised exactly to F = rint(f * 2^16)
// (|F / 2^16 - f_ref| <= E + 2^-17, E the certified sample bound), so the
// window sums sum F, sum F^2 and sum r*F are EXACT integers and can be formed
// as separable box sums: one thread per (view, tile column, half column)
// slides a WW x WH window down 4 pixel rows (WH + 3 row sums instead of 4 x WH).
// From the exact quantised var_q and cov_q the reference's FP64 values are
// bracketed rigorously: the centred sample vector moves by at most
// ||e|| <= sqrt(n) * e_max, so sqrt(var) moves by at most ||e|| (centring is
// an orthogonal projection) and cov by at most sqrt(ref_var) * ||e||
// (Cauchy-Schwarz); the reference's own FP64 rounding (< 1e-7 absolute) is
// covered by requiring var_q >= 1 and the relative slack of the FP32 bound
// arithmetic. When both ends of 255*min(1 - ncc, 1) round to the same
// integer the cost is certified; otherwise the whole window is recomputed
// with the reference's exact FP64 walk (NS work items, one sample per thread)
// and the reference's exact sum order.
// ===================================================================

constexpr int kNccItemCap = 2048;
constexpr int kNccPend = 128;  // pending (pixel, plane) entries per batch

// sqrt(x) for bounds: MUFU rsqrt based (relative error < 1e-6), 0 for x <= 0.
__device__ __forceinline__ float sqrt_up(float x) { return x > 0.0f ? x * rsqrtf(x) * 1.0001f : 0.0f; }

// The tail of the reference's NCC cost from its FP64 window sums
// (matching.cpp:271-279).
template <int NS>
__device__ __forceinline__ int ncc_tail(double sb, double sbb, double sab, double ref_mean,
                                        double ref_var) {
    using namespace dev;
    const double var_b = sub(sbb, div(mul(sb, sb), double(NS)));
    if (var_b <= 0.0)
        return 255;
    const double ncc = div(sub(sab, mul(ref_mean, sb)), sqrt_(mul(ref_var, var_b)));
    const double t = sub(1.0, ncc);
    double cc = mul(255.0, 1.0 < t ? 1.0 : t);
    cc = cc < 0.0 ? 0.0 : (255.0 < cc ? 255.0 : cc);
    return static_cast<int>(lround(cc));
}

// Exact FP64 NCC cost of one view (tile certification impossible; rare), out
// of line so its registers do not weigh on the tiled kernel. `ref` points at
// the pixel's window in the shared reference tile (row stride `sw`).
template <int WW, int WH>
__device__ __noinline__ int ncc_view_exact(const uint32_t* __restrict__ quad, int vw, int vh,
                                           const double* __restrict__ hp, double xd, double yd,
                                           const int* ref, int sw, double ref_mean, double ref_var,
                                           const uint16_t* __restrict__ lut) {
    float patch[WW * WH];
    for (int i = 0; i < WH; ++i)
        for (int j = 0; j < WW; ++j)
            patch[i * WW + j] = float(ref[i * sw + j]);
    return view_cost<FMVS_COST_NCC, WW, WH>(quad, vw, vh, hp, xd, yd, 0ull, patch, ref_mean, ref_var, lut);
}

// Exact integer window sums of the quantised samples (see the header above).
struct NccSums {
    uint32_t f;   // sum F            < NS * 2^24
    uint64_t ff;  // sum F^2          < NS * 2^48
    uint64_t rf;  // sum r * F        < NS * 2^32
};

// Certified NCC cost of one window from its exact sums, or -1.
//   var_q = (n SF^2 - (SF)^2) / (n 2^32), cov_q = (n SrF - Sr SF) / (n 2^16)
// are the quantised window's exact centred sums (FP32-rounded: < 2e-7 rel.).
// The reference's sqrt(var_b) lies within D = e_norm + 1e-6 sv of
// sv = sqrt(var_q) and its covariance within dc of cov_q, so its ncc lies
// within  dn = (dc + |n| rho D) / (rho (sv - D))  of n = cov_q / (rho sv);
// with D <= sv/128, 1/(sv - D) <= 1.01/sv. The cost 255 min(1 - ncc, 1)
// clamped to [0, 255] is monotone and 255-Lipschitz in ncc, so if both ends
// of its interval round (half up) to the same integer that is the
// reference's cost.
template <int NS>
__device__ __forceinline__ int ncc_certify(const NccSums& S, int rsum, float rho, float e_norm) {
    // n^2 * var_q * 2^32 and n * cov_q * 2^16, exact
    const long long nv = static_cast<long long>(NS) * static_cast<long long>(S.ff) -
                         static_cast<long long>(static_cast<unsigned long long>(S.f) * S.f);
    const long long nc = static_cast<long long>(NS) * static_cast<long long>(S.rf) -
                         static_cast<long long>(rsum) * static_cast<long long>(S.f);
    constexpr float inv_nv = 1.0f / (float(NS) * 4294967296.0f);  // relative error < 1e-7
    constexpr float inv_nc = 1.0f / (float(NS) * 65536.0f);
    const float var_q = float(nv) * inv_nv;
    const float sv = var_q * rsqrtf(var_q);  // sqrt(var_q), rel. error < 4e-7 (NaN if var_q <= 0)
    const float D = fmaf(sv, 1.0e-6f, e_norm);
    // var_q >= 1: near-flat windows, where the reference's FP64 rounding is
    // not negligible, are left to the exact walk
    if (!(var_q >= 1.0f) || !(128.0f * D <= sv))
        return -1;
    const float c_q = float(nc) * inv_nc;
    const float dc = fmaf(rho, e_norm, fmaf(fabsf(c_q), 1.0e-6f, 1.0e-6f));
    float inv;  // 1/(rho sv): MUFU reciprocal, rel. error < 2^-22 (in the slack)
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(rho * sv));
    const float n = c_q * inv;
    // FP32 bound arithmetic (conversions, products, MUFU rsqrt / rcp; < 1e-6
    // rel.) and the reference's FP64 rounding (< 1e-7 abs. with var >= 1)
    const float dn = fmaf(fmaf(fabsf(n) * rho, D, dc), inv * 1.01f, fmaf(fabsf(n), 4.0e-6f, 2.0e-6f));
    const float t = fminf(fmaxf(255.0f * fminf(1.0f - n, 1.0f), 0.0f), 255.0f) + 0.5f;
    const float w = fmaf(255.0f, dn, 2.0e-4f);
    const int k_lo = static_cast<int>(floorf(t - w));
    const int k_hi = static_cast<int>(floorf(t + w));
    return k_lo == k_hi ? k_lo : -1;
}

// TH: tile height (8: 256 threads; 16: 512 threads, fewer halo samples per
// pixel: 36 x 20 / 512 = 1.41 instead of 36 x 12 / 256 = 1.69)
template <int WW, int WH, int NM, int TH>
__global__ void __launch_bounds__(32 * TH, TH == 16 ? 2 : FMVS_NCC_MINB_OF(WW * WH, NM))
    sweep_ncc_tiled(SweepArgs a) {
    using namespace dev;
    constexpr int NT = kTW * TH;           // threads = tile pixels
    constexpr int TB = NT > 256 ? 9 : 8;   // bits of a thread index in the item / pending words
    constexpr uint32_t TM = (1u << TB) - 1;
    constexpr int RX = WW / 2, RY = WH / 2, NS = WW * WH;
    constexpr int SW = kTW + WW - 1, SH = TH + WH - 1, SN = SW * SH;
    constexpr int kRows = 4;                       // pixel rows per box-sum thread
    constexpr int kQ = TH / kRows;                 // box-sum row groups per column
    static_assert(TH == kQ * kRows, "box-sum thread map");
    extern __shared__ int s_F[];  // [NM][SH][SW] quantised samples F = rint(f * 2^16)
    // certified cost per (view, pixel) or -1, then the certified inside flag
    // of each tile sample as a window centre (general tiles only)
    int16_t* s_cost = reinterpret_cast<int16_t*>(s_F + NM * SN);  // [NM][NT]
    uint8_t* s_in = reinterpret_cast<uint8_t*>(s_cost + NM * NT);
    // dense levels: staged runs (after the inside flags, 16-byte aligned)
    uint16_t* s_run = reinterpret_cast<uint16_t*>(
        (reinterpret_cast<uintptr_t>(s_in + NM * SN) + 15) & ~static_cast<uintptr_t>(15));
    __shared__ int s_ref[SN];  // edge-clamped reference tile + halo (u8 values)
    __shared__ TileParams64 s_tp[kPlaneChunk][NM];
    __shared__ ViewConst s_vc[NM];
    __shared__ int s_pmin, s_pmax;
    __shared__ int s_count;  // exact samples listed for the current batch of planes
    __shared__ int s_npend;  // pending (pixel, plane) entries of the batch
    // max sample bound of the tile (float bits), by plane parity: reset for
    // plane p + 1 between barriers T and C of plane p
    __shared__ unsigned s_emax[2][NM];
    __shared__ int s_rsum[NT];            // sum r of each pixel's window
    __shared__ float s_rho[NT];           // sqrt(ref_var), 0 if ref_var <= 0
    __shared__ uint32_t s_items[kNccItemCap];        // t | m << TB | pos << TB+4 | slot << TB+11
    __shared__ double s_vals[kNccItemCap];
    // (sum_l | sum_r << 16, t | slot << TB | undecided views << TB+3 | first view index << TB+11)
    __shared__ uint2 s_pend[kNccPend];
    int* s_first = reinterpret_cast<int*>(s_vals);  // prologue only (aliases s_vals)
    int* s_cnt = s_first + NT;
    __shared__ int s_vcost[kNccItemCap / NS + 1];  // pass 2b results
    __shared__ double s_rmean[NT], s_rvar[NT];
    constexpr int kTPV = NT / NM;
    // capacities of the exact lists (the test hook shrinks them)
    const int icap = a.small_lists ? 2 * NS : kNccItemCap;
    const int pcap = a.small_lists ? 2 : kNccPend;  // tile-build threads per view

    const int tx = threadIdx.x % kTW, ty = threadIdx.x / kTW;
    const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * TH;
    const int x = x0 + tx, y = y0 + ty;
    const bool in_img = x < a.w && y < a.h;

    for (int r = threadIdx.x; r < SN; r += NT) {
        const int dv = r / SW, du = r - dv * SW;
        const int xx = min(max(x0 - RX + du, 0), a.w - 1);
        const int yy = min(max(y0 - RY + dv, 0), a.h - 1);
        s_ref[r] = a.ref_img[static_cast<size_t>(yy) * a.w + xx];
    }
    int first = 0, count = 0;
    uint64_t base = 0;
    if (in_img) {
        const VolMeta m = a.meta[static_cast<size_t>(y) * a.w + x];
        first = meta_first(m.fc);
        count = meta_count(m.fc);
        base = a.row_base[y] + m.rel;
        if (count > a.exact_above)
            count = 0;  // wide pixel: the exact per-hypothesis kernel owns it
    }
    s_first[threadIdx.x] = first;
    s_cnt[threadIdx.x] = count;
    if (threadIdx.x == 0) {
        s_pmin = 0x7FFFFFFF;
        s_pmax = -1;
        s_count = 0;
        s_npend = 0;
    }
    if (threadIdx.x < NM) {
        const int m = threadIdx.x;
        const int2 sz = a.sizes[m];
        s_vc[m] = ViewConst{a.quads[m], a.homs + static_cast<size_t>(m) * a.nplanes * 9, sz.x, sz.y,
                            m < a.nleft ? 1 : 0};
        s_emax[0][m] = 0u;
        s_emax[1][m] = 0u;
    }
    __syncthreads();
    // reference patch mean and two-pass variance, exactly as matching.cpp:199-210
    double ref_mean = 0.0, ref_var = 0.0;
    int rsum = 0;
    if (count > 0) {
#pragma unroll
        for (int i = 0; i < WH; ++i)
#pragma unroll
            for (int j = 0; j < WW; ++j) {
                const int r = s_ref[(ty + i) * SW + tx + j];
                ref_mean = add(ref_mean, double(r));
                rsum += r;
            }
        ref_mean = div(ref_mean, double(NS));
#pragma unroll
        for (int i = 0; i < WH; ++i)
#pragma unroll
            for (int j = 0; j < WW; ++j) {
                const double d = sub(double(s_ref[(ty + i) * SW + tx + j]), ref_mean);
                ref_var = add(ref_var, mul(d, d));
            }
        s_rmean[threadIdx.x] = ref_mean;
        s_rvar[threadIdx.x] = ref_var;
        atomicMin(&s_pmin, first);
        atomicMax(&s_pmax, first + count - 1);
    }
    s_rsum[threadIdx.x] = rsum;
    // sqrt(ref_var) rounded down (|rel. error| of the FP32 path < 1e-6 is in
    // the certification slack)
    s_rho[threadIdx.x] = ref_var > 0.0 ? __double2float_rd(sqrt_(ref_var)) : 0.0f;
    __syncthreads();
    const int slice = (a.nplanes + gridDim.z - 1) / gridDim.z;
    const int pmin = max(s_pmin, static_cast<int>(blockIdx.z) * slice);
    const int pmax = min(s_pmax, static_cast<int>(blockIdx.z + 1) * slice - 1);
    const double xd = double(x), yd = double(y);
    // plane union of the 4 pixels of each box-sum job this thread serves
    constexpr int kJobs = (NM * kQ * kTW + NT - 1) / NT;
    int job_lo[kJobs], job_hi[kJobs];
#pragma unroll
    for (int jj = 0; jj < kJobs; ++jj) {
        const int job = threadIdx.x + jj * NT;
        const int bc = job % kTW, bh = (job / kTW) % kQ;
        job_lo[jj] = 0x7FFFFFFF;
        job_hi[jj] = -1;
#pragma unroll
        for (int k = 0; k < kRows; ++k) {
            const int pix = (bh * kRows + k) * kTW + bc;
            if (s_cnt[pix] > 0) {
                job_lo[jj] = min(job_lo[jj], s_first[pix]);
                job_hi[jj] = max(job_hi[jj], s_first[pix] + s_cnt[pix] - 1);
            }
        }
    }

    for (int p = pmin; p <= pmax; ++p) {
        const bool need = count > 0 && p >= first && p < first + count;
        const int slot = (p - pmin) % kPlaneChunk;
        if (slot == 0) {
            // tile parameters of the next kPlaneChunk planes x NM views (the
            // previous chunk's were last read in the box pass of the previous
            // plane, before its barrier C)
            for (int k = threadIdx.x; k < kPlaneChunk * NM; k += NT) {
                const int pp = p + k / NM, m = k % NM;
                if (pp <= pmax)
                    s_tp[k / NM][m] = make_tile_params64(s_vc[m].homs + static_cast<size_t>(pp) * 9,
                                                         x0 - RX, y0 - RY, SW - 1, SH - 1, s_vc[m].w,
                                                         s_vc[m].h);
            }
            __syncthreads();
        }
        // Two barriers per plane: tile complete (T), box costs complete (C);
        // at the end of each run of kRunNcc planes (or earlier when the lists
        // fill up): exact-sample lists complete (I), exact samples taken (P),
        // view costs resolved (B) and, on dense levels, the staged run
        // complete (R).
        // ---- tile build: each thread serves one view (parameters in
        // registers); quantised samples, the tile's max sample bound
        if (threadIdx.x < NM * kTPV) {
            const int m = threadIdx.x / kTPV;
            const TileParams64 tp = s_tp[slot][m];
            const ViewConst vc = s_vc[m];
            int* t = s_F + m * SN;
            uint8_t* fl = s_in + m * SN;
            const int r = threadIdx.x - m * kTPV;
            float emax = 0.0f;
            if (tp.exact != kTileExact)
                emax = tp.eb > 0.0f ? build_ncc_tile<false, SW, SN, kTPV>(tp, vc, t, fl, r)
                                    : build_ncc_tile<true, SW, SN, kTPV>(tp, vc, t, fl, r);
            // tile maximum of the bounds (positive floats: their bit patterns
            // order like them); lanes of one warp may serve different views
            const unsigned grp = __match_any_sync(__activemask(), m);
            const unsigned eb = __reduce_max_sync(grp, __float_as_uint(emax));
            if ((threadIdx.x & 31) == __ffs(grp) - 1)
                atomicMax(&s_emax[p & 1][m], eb);
        }
        __syncthreads();  // T
        if (threadIdx.x < NM)
            s_emax[(p + 1) & 1][threadIdx.x] = 0u;
        // per-view flags of this pixel for pass 1 (s_tp and s_in are rewritten
        // by the next planes before pass 1 of this one may run)
        const int bslot = (p - pmin) % kRunNcc;  // plane's slot in its run
        // lists already half full (appended by planes < p, reset before T):
        // resolve at the end of this plane instead of the run's end
        const bool early = s_count >= icap / 2 || s_npend >= pcap / 2;
        uint32_t view_in = 0, view_exact = 0;
        if (need) {
#pragma unroll
            for (int m = 0; m < NM; ++m) {
                const int tpe = s_tp[slot][m].exact;
                if (tpe == kTileExact) {
                    view_exact |= 1u << m;
                } else if (tpe == kTileInterior) {
                    view_in |= 1u << m;
                } else {
                    const uint8_t fl = s_in[m * SN + (ty + RY) * SW + tx + RX];
                    if (fl == 2 ? exact_inside(s_vc[m].homs + static_cast<size_t>(p) * 9, s_vc[m].w, s_vc[m].h,
                                               double(x), double(y))
                                : fl == 1)
                        view_in |= 1u << m;
                }
            }
        }
        // ---- box pass: exact window sums by sliding row sums, certified cost
        // per (view, pixel) into s_cost; job = (view m, tile column bc,
        // pixel rows bh*4 .. bh*4+3)
#pragma unroll
        for (int jj = 0; jj < kJobs; ++jj) {
            const int job = threadIdx.x + jj * NT;
            if (job >= NM * kQ * kTW)
                break;
            const int m = job / (kQ * kTW), bc = job % kTW, bh = (job / kTW) % kQ;
            const int tpe = s_tp[slot][m].exact;
            // (a pixel of the job needing another plane inside the union
            // only costs a wasted certification)
            if (tpe != kTileExact && p >= job_lo[jj] && p <= job_hi[jj]) {
                const int* F = s_F + m * SN;
                // ||e|| <= sqrt(n) * (E_max + 2^-17), rounded up
                const float e_norm =
                    sqrtf(float(NS)) * (__uint_as_float(s_emax[p & 1][m]) + 7.7e-6f) * 1.0001f;
                auto row_sum = [&](int row) {
                    NccSums R{0u, 0ull, 0ull};
#pragma unroll
                    for (int j = 0; j < WW; ++j) {
                        const uint32_t f = static_cast<uint32_t>(F[row * SW + bc + j]);
                        const uint32_t rv = static_cast<uint32_t>(s_ref[row * SW + bc + j]);
                        R.f += f;
                        R.ff += static_cast<uint64_t>(f) * f;
                        R.rf += static_cast<uint64_t>(rv) * f;
                    }
                    return R;
                };
                const int row0 = bh * kRows;
                NccSums S{0u, 0ull, 0ull}, keep[kRows - 1];
#pragma unroll
                for (int i = 0; i < WH; ++i) {
                    const NccSums R = row_sum(row0 + i);
                    if (i < kRows - 1)
                        keep[i] = R;
                    S.f += R.f;
                    S.ff += R.ff;
                    S.rf += R.rf;
                }
#pragma unroll
                for (int k = 0; k < kRows; ++k) {
                    if (k > 0) {
                        const NccSums R = row_sum(row0 + k - 1 + WH);
                        S.f += R.f - keep[k - 1].f;
                        S.ff += R.ff - keep[k - 1].ff;
                        S.rf += R.rf - keep[k - 1].rf;
                    }
                    const int pix = (row0 + k) * kTW + bc;
                    const float rho = s_rho[pix];
                    s_cost[m * NT + pix] = static_cast<int16_t>(
                        rho > 0.0f ? ncc_certify<NS>(S, s_rsum[pix], rho, e_norm) : -1);
                }
            }
        }
        __syncthreads();  // C
        // ---- pass 1: per-side sums of the certified costs. Pixels with
        // undecided views list NS exact work items per view and a pending
        // entry; the exact samples of a whole batch of planes (a staged run)
        // are taken and resolved together at its end.
        if (need) {
            int sum_l = 0, sum_r = 0, nun = 0;
            uint32_t unsure = 0;
            const bool flat = !(s_rho[threadIdx.x] > 0.0f);  // ref_var <= 0
#pragma unroll
            for (int m = 0; m < NM; ++m) {
                int c = 255;  // outside / flat reference (matching.cpp:224-232, 262-263)
                if ((view_exact >> m) & 1u) {
                    c = ncc_view_exact<WW, WH>(s_vc[m].quad, s_vc[m].w, s_vc[m].h,
                                               s_vc[m].homs + static_cast<size_t>(p) * 9, double(x), double(y),
                                               s_ref + ty * SW + tx, SW, s_rmean[threadIdx.x],
                                               s_rvar[threadIdx.x], a.census_lut);
                } else if (((view_in >> m) & 1u) && !flat) {
                    c = s_cost[m * NT + threadIdx.x];
                    if (a.stats) {
                        atomicAdd(a.stats + 0, 1ull);
                        if (c < 0)
                            atomicAdd(a.stats + 1, 1ull);
                    }
                    if (c < 0) {
                        unsure |= 1u << m;
                        ++nun;
                        c = 0;
                    }
                }
                if (m < a.nleft)
                    sum_l += c;
                else
                    sum_r += c;
            }
            bool done = unsure == 0;
            if (!done) {
                const int e = atomicAdd(&s_npend, 1);
                const int off = e < pcap ? atomicAdd(&s_count, nun * NS) : icap;
                const uint32_t tag = threadIdx.x | (bslot << (TB + 11));
                if (off + nun * NS <= icap) {
                    int k = off;
                    for (uint32_t u = unsure; u; u &= u - 1) {
                        const uint32_t mt = tag | ((__ffs(u) - 1) << TB);
                        for (int q = 0; q < NS; ++q)
                            s_items[k++] = mt | (q << (TB + 4));
                    }
                    s_pend[e] = make_uint2(static_cast<uint32_t>(sum_l) | (static_cast<uint32_t>(sum_r) << 16),
                                           threadIdx.x | (bslot << TB) | (unsure << (TB + 3)) |
                                               (static_cast<uint32_t>(off / NS) << (TB + 11)));
                } else {
                    // list overflow (pathological inputs): the owner walks its
                    // views; reserved slots get harmless dummy items
                    if (e < pcap) {
                        for (int k = off; k < min(off + nun * NS, icap); ++k)
                            s_items[k] = tag | ((__ffs(unsure) - 1) << TB);
                        s_pend[e] = make_uint2(0u, 0xFFFFFFFFu);
                    }
                    for (uint32_t u = unsure; u; u &= u - 1) {
                        const int m = __ffs(u) - 1;
                        const ViewConst& vc = s_vc[m];
                        const double* hp = vc.homs + static_cast<size_t>(p) * 9;
                        double sb = 0.0, sbb = 0.0, sab = 0.0;
                        for (int q = 0; q < NS; ++q) {
                            const int i = q / WW, j = q - (q / WW) * WW;
                            const double v = exact_window_sample(hp, vc.quad, vc.w, vc.h, double(x), double(y),
                                                                 RX, RY, i, j);
                            sb = add(sb, v);
                            sbb = add(sbb, mul(v, v));
                            sab = add(sab, mul(double(s_ref[(ty + i) * SW + tx + j]), v));
                        }
                        const int c = ncc_tail<NS>(sb, sbb, sab, s_rmean[threadIdx.x], s_rvar[threadIdx.x]);
                        if (m < a.nleft)
                            sum_l += c;
                        else
                            sum_r += c;
                    }
                    done = true;
                }
            }
            if (done) {
                const uint16_t v = static_cast<uint16_t>(min(sum_l, sum_r));
                if (a.plane_slicing)
                    s_run[threadIdx.x * (kRunNcc + 2) + bslot] = v;
                else
                    a.costs[base + static_cast<uint64_t>(p - first)] = v;
            }
        }
        const bool run_end = bslot == kRunNcc - 1 || p == pmax;
        if (run_end || early) {
            const int pb = p - bslot;  // first plane of the run
            __syncthreads();  // I: item and pending lists complete
            const int total = s_count;
            const int npend = min(s_npend, pcap);
            const int nitems = min(total, icap);
            if (a.stats && threadIdx.x == 0)
                atomicAdd(a.stats + 6, static_cast<unsigned long long>(total));
            // ---- pass 2: the exact samples, one per thread
            for (int it = threadIdx.x; it < nitems; it += NT) {
                const uint32_t item = s_items[it];
                const int t = item & TM, m = (item >> TB) & 0xF, pos = (item >> (TB + 4)) & 0x7F;
                const ViewConst& vc = s_vc[m];
                s_vals[it] = exact_window_sample(vc.homs + static_cast<size_t>(pb + (item >> (TB + 11))) * 9, vc.quad,
                                                 vc.w, vc.h, double(x0 + t % kTW), double(y0 + t / kTW), RX, RY,
                                                 pos / WW, pos % WW);
            }
            __syncthreads();  // P
            if (threadIdx.x == 0) {
                s_count = 0;  // read by every thread before P; next appended after C
                s_npend = 0;
            }
            // ---- pass 2b: the reference's sums and NCC of each undecided view
            // (matching.cpp:265-279, same order), one thread per view
            const int nviews_u = nitems / NS;
            for (int v = threadIdx.x; v < nviews_u; v += NT) {
                const int k0 = v * NS;
                const int t = s_items[k0] & TM;
                const int ttx = t % kTW, tty = t / kTW;
                double sb = 0.0, sbb = 0.0, sab = 0.0;
                for (int q = 0; q < NS; ++q) {
                    const int i = q / WW, j = q - (q / WW) * WW;
                    const double val = s_vals[k0 + q];
                    sb = add(sb, val);
                    sbb = add(sbb, mul(val, val));
                    sab = add(sab, mul(double(s_ref[(tty + i) * SW + ttx + j]), val));
                }
                s_vcost[v] = ncc_tail<NS>(sb, sbb, sab, s_rmean[t], s_rvar[t]);
            }
            __syncthreads();  // B
            // ---- pass 3: pending entries -> final costs
            for (int e = threadIdx.x; e < npend; e += NT) {
                const uint2 pe = s_pend[e];
                if (pe.y == 0xFFFFFFFFu)
                    continue;
                const int t = pe.y & TM, sl = (pe.y >> TB) & 7;
                int vi = static_cast<int>(pe.y >> (TB + 11));
                int sum_l = static_cast<int>(pe.x & 0xFFFFu), sum_r = static_cast<int>(pe.x >> 16);
                for (uint32_t u = (pe.y >> (TB + 3)) & 0xFFu; u; u &= u - 1) {
                    const int c = s_vcost[vi++];
                    if (__ffs(u) - 1 < a.nleft)
                        sum_l += c;
                    else
                        sum_r += c;
                }
                const uint16_t v = static_cast<uint16_t>(min(sum_l, sum_r));
                if (a.plane_slicing) {
                    s_run[t * (kRunNcc + 2) + sl] = v;
                } else {
                    const int xt = x0 + t % kTW, yt = y0 + t / kTW;
                    const VolMeta mt = a.meta[static_cast<size_t>(yt) * a.w + xt];
                    a.costs[a.row_base[yt] + mt.rel + static_cast<uint64_t>(pb + sl - meta_first(mt.fc))] = v;
                }
            }
            if (a.plane_slicing && run_end) {
                __syncthreads();  // R: the run is complete
                flush_run<kRunNcc>(a.costs, s_run + threadIdx.x * (kRunNcc + 2), pb, p, first, count, base);
            }
        }
    }
}

template <int WW, int WH, int NM, int TH>
void launch_ncc_nm(const SweepArgs& a, int slices, cudaStream_t s) {
    constexpr int NT = kTW * TH;
    const size_t smem = (sizeof(int) + 1) * NM * (kTW + WW - 1) * (TH + WH - 1) +
                        sizeof(int16_t) * NM * NT + 16 +
                        (a.plane_slicing ? sizeof(uint16_t) * NT * (kRunNcc + 2) : 0);
    // attribute: the largest size (with the dense-level run staging), a
    // constant -- contexts on other host threads launch the same kernel
    const int smem_max = static_cast<int>((sizeof(int) + 1) * NM * (kTW + WW - 1) * (TH + WH - 1) +
                                          sizeof(int16_t) * NM * NT + 16 +
                                          sizeof(uint16_t) * NT * (kRunNcc + 2));
    FMVS_CUDA_CHECK(cudaFuncSetAttribute(sweep_ncc_tiled<WW, WH, NM, TH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    const dim3 grid((a.w + kTW - 1) / kTW, (a.h + TH - 1) / TH, slices);
    sweep_ncc_tiled<WW, WH, NM, TH><<<grid, NT, smem, s>>>(a);
}

// Dense levels (every pixel sweeps the whole stack) with 5x5 windows and <= 4
// matching views use 32 x 16 tiles (512 threads, 2 CTAs per SM at 64
// registers; same threads per slice). Refined levels keep 32 x 8: a taller
// tile widens the plane union its pixels iterate (measured: C2-NCC L0 1.98
// -> 2.25 ms with 32 x 16). 9x9 windows and more views: their register budgets.
template <int WW, int WH>
bool launch_ncc(const SweepArgs& a, int slices, cudaStream_t s) {
    const bool tall = WW * WH == 25 && a.plane_slicing;
    switch (a.nmatch) {
        case 2:
            if (tall)
                launch_ncc_nm<WW, WH, 2, 16>(a, slices, s);
            else
                launch_ncc_nm<WW, WH, 2, 8>(a, slices, s);
            return true;
        case 4:
            if (tall)
                launch_ncc_nm<WW, WH, 4, 16>(a, slices, s);
            else
                launch_ncc_nm<WW, WH, 4, 8>(a, slices, s);
            return true;
        case 6: launch_ncc_nm<WW, WH, 6, 8>(a, slices, s); return true;
        case 8: launch_ncc_nm<WW, WH, 8, 8>(a, slices, s); return true;
        default: return false;
    }
}

template <int WW, int WH, int NM>
void launch_tiled_nm(const SweepArgs& a, dim3 grid, cudaStream_t s) {
    const size_t smem = sizeof(float2) * NM * (kTW + WW - 1) * (kTH + WH - 1);
    FMVS_CUDA_CHECK(cudaFuncSetAttribute(sweep_census_tiled<WW, WH, NM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
    sweep_census_tiled<WW, WH, NM><<<grid, kTiledThreads, smem, s>>>(a);
}

template <int WW, int WH>
bool launch_tiled(const SweepArgs& a, dim3 grid, cudaStream_t s) {
    switch (a.nmatch) {
        case 2: launch_tiled_nm<WW, WH, 2>(a, grid, s); return true;
        case 4: launch_tiled_nm<WW, WH, 4>(a, grid, s); return true;
        case 6: launch_tiled_nm<WW, WH, 6>(a, grid, s); return true;
        case 8: launch_tiled_nm<WW, WH, 8>(a, grid, s); return true;
        default: return false;
    }
}

}  // namespace

int sweep(const SweepArgs& a_in, cudaStream_t s) {
    SweepArgs a = a_in;
    const bool tiled = !a.disable_tiled &&
                       (a.nmatch == 2 || a.nmatch == 4 || a.nmatch == 6 || a.nmatch == 8);
    // Pixels wider than narrow_max (invalid-prior pixels sweeping the whole
    // stack at refined levels) would inflate a tile's plane union: they take
    // the exact per-hypothesis kernel. Uniform levels set narrow_max to the
    // stack size (every pixel shares the range).
    a.exact_above = tiled ? (a.narrow_max > 0 ? a.narrow_max : kNarrowMax) : 0;
    const int nseg = ((a.w + kSeg - 1) / kSeg) * a.h;
    const dim3 grid(std::max(1, std::min(nseg, 148 * 16)));
    if (a.kind == FMVS_COST_CENSUS && a.ww == 5)
        sweep_kernel<FMVS_COST_CENSUS, 5, 5><<<grid, kThreads, 0, s>>>(a);
    else if (a.kind == FMVS_COST_CENSUS)
        sweep_kernel<FMVS_COST_CENSUS, 9, 7><<<grid, kThreads, 0, s>>>(a);
    else if (a.ww == 5)
        sweep_kernel<FMVS_COST_NCC, 5, 5><<<grid, kThreads, 0, s>>>(a);
    else
        sweep_kernel<FMVS_COST_NCC, 9, 9><<<grid, kThreads, 0, s>>>(a);
    FMVS_CUDA_CHECK(cudaGetLastError());
    if (!tiled)
        return 1;
    // Dense levels with few tiles: split the plane range across gridDim.z so
    // the launch covers >= ~4 waves of 148 SMs x 3 CTAs.
    const int tiles = ((a.w + kTW - 1) / kTW) * ((a.h + kTH - 1) / kTH);
    int slices = 1;
#ifndef FMVS_SLICE_TARGET
// measured on C2 L2 (510 tiles): 2 slices 179.4 maps/s, 4 slices 180.8, 8
// slices 179.7 (lower single-bundle latency, more per-CTA prologues)
#define FMVS_SLICE_TARGET (4 * 148 * 3)
#endif
    if (a.plane_slicing)
        while (slices < 64 && tiles * slices < FMVS_SLICE_TARGET && a.nplanes / (2 * slices) >= 8)
            slices *= 2;
    const dim3 tgrid((a.w + kTW - 1) / kTW, (a.h + kTH - 1) / kTH, slices);
    if (a.kind == FMVS_COST_CENSUS && a.ww == 5)
        launch_tiled<5, 5>(a, tgrid, s);
    else if (a.kind == FMVS_COST_CENSUS)
        launch_tiled<9, 7>(a, tgrid, s);
    else if (a.ww == 5)
        launch_ncc<5, 5>(a, slices, s);
    else
        launch_ncc<9, 9>(a, slices, s);
    FMVS_CUDA_CHECK(cudaGetLastError());
    return 2;  // exact (wide pixels) + tiled
}

}  // namespace k
}  // namespace fmvs
