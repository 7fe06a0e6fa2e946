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
    __shared__ int s_prefix[kSeg + 1];
    __shared__ int s_first[kSeg];
    __shared__ uint64_t s_bits[kSeg];
    __shared__ double s_mean[kSeg], s_var[kSeg];
    __shared__ float s_patch[kSeg][NSP];
    __shared__ uint64_t s_base;

    const int y = blockIdx.y;
    const int x0 = blockIdx.x * kSeg;
    const int npx = min(kSeg, a.w - x0);
    const int t = threadIdx.x;
    const uint8_t* ref = a.ref_img;

    if (t < 32) {
        int cnt = 0;
        if (t < npx) {
            const VolMeta m = a.meta[static_cast<size_t>(y) * a.w + x0 + t];
            cnt = meta_count(m.fc);
            s_first[t] = meta_first(m.fc);
            if (t == 0)
                s_base = a.row_base[y] + m.rel;
        }
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (t >= o)
                incl += v;
        }
        s_prefix[t + 1] = incl;
        if (t == 0)
            s_prefix[0] = 0;
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
                s_bits[t] = bits;
            } else {
                // reference patch, mean and two-pass variance (matching.cpp:199-210)
                int s = 0;
                for (int dy = -RY; dy <= RY; ++dy)
                    for (int dx = -RX; dx <= RX; ++dx) {
                        const int xx = min(max(x + dx, 0), a.w - 1);
                        const int yy = min(max(y + dy, 0), a.h - 1);
                        s_patch[t][s++] = float(ref[static_cast<size_t>(yy) * a.w + xx]);
                    }
                double mean = 0.0, var = 0.0;
                for (int i = 0; i < NS; ++i)
                    mean = add(mean, double(s_patch[t][i]));
                mean = div(mean, double(NS));
                for (int i = 0; i < NS; ++i) {
                    const double d = sub(double(s_patch[t][i]), mean);
                    var = add(var, mul(d, d));
                }
                s_mean[t] = mean;
                s_var[t] = var;
            }
        }
    }
    __syncthreads();

    const int total = s_prefix[npx];
    const uint64_t base = s_base;
    for (int e = t; e < total; e += kThreads) {
        // pixel of entry e: largest j with prefix[j] <= e
        int lo = 0, hi = npx;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_prefix[mid] <= e)
                lo = mid;
            else
                hi = mid;
        }
        const int j = lo;
        const int plane = s_first[j] + (e - s_prefix[j]);
        const double xd = double(x0 + j), yd = double(y);
        int sum_l = 0, sum_r = 0;
        for (int m = 0; m < a.nmatch; ++m) {
            const int2 sz = a.sizes[m];
            const int c = view_cost<KIND, WW, WH>(
                a.quads[m], sz.x, sz.y, a.homs + (static_cast<size_t>(m) * a.nplanes + plane) * 9,
                xd, yd, KIND == FMVS_COST_CENSUS ? s_bits[j] : 0ull,
                KIND == FMVS_COST_NCC ? s_patch[j] : nullptr,
                KIND == FMVS_COST_NCC ? s_mean[j] : 0.0, KIND == FMVS_COST_NCC ? s_var[j] : 0.0,
                a.census_lut);
            if (m < a.nleft)
                sum_l += c;
            else
                sum_r += c;
        }
        a.costs[base + e] = static_cast<uint16_t>(min(sum_l, sum_r));
        if (a.agg_zero)
            a.agg_zero[base + e] = 0u;
    }
}

}  // namespace

void sweep(const SweepArgs& a, cudaStream_t s) {
    const dim3 grid((a.w + kSeg - 1) / kSeg, a.h);
    if (a.kind == FMVS_COST_CENSUS && a.ww == 5)
        sweep_kernel<FMVS_COST_CENSUS, 5, 5><<<grid, kThreads, 0, s>>>(a);
    else if (a.kind == FMVS_COST_CENSUS)
        sweep_kernel<FMVS_COST_CENSUS, 9, 7><<<grid, kThreads, 0, s>>>(a);
    else if (a.ww == 5)
        sweep_kernel<FMVS_COST_NCC, 5, 5><<<grid, kThreads, 0, s>>>(a);
    else
        sweep_kernel<FMVS_COST_NCC, 9, 9><<<grid, kThreads, 0, s>>>(a);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

}  // namespace k
}  // namespace fmvs
