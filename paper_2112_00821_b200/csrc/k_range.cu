// K3: per-pixel sampling range, plane interval and the ragged-volume layout.
//
// One CTA per image row. Each pixel evaluates
//   - its sampling range: uniform (SamplingRange::uniform, matching.cpp:20-26)
//     or refine_range of the upscaled prior (pipeline.cpp:136-173, with the
//     nearest-neighbour upscale of pipeline.cpp:91-103 folded into the read),
//     stored as float exactly like the reference's Raster<float>;
//   - its plane interval [first, last] (plane_interval, matching.cpp:95-107),
//     found by two binary searches instead of the reference's linear scans
//     (valid because scale*delta_i is monotone in i under round-to-nearest);
// then the row's counts are exclusive-scanned into row-relative offsets.
// scan_rows turns the per-row totals into 64-bit row bases, so the whole
// layout is produced on device with no host synchronisation.
#include <cub/block/block_scan.cuh>

#include "host.hpp"
#include "kernels.hpp"

namespace fmvs {
namespace k {

namespace {

constexpr int kRangeThreads = 256;

__device__ __forceinline__ void pixel_range(const RangeArgs& a, int x, int y, float* lo_f,
                                            float* hi_f) {
    using namespace dev;
    float lo = __double2float_rn(a.d_min);
    float hi = __double2float_rn(a.d_max);
    if (a.mode == 2) {
        const size_t p = static_cast<size_t>(y) * a.intr.w + x;
        lo = a.lo_in[p];
        hi = a.hi_in[p];
    } else if (a.mode == 1 && a.policy != FMVS_RANGE_FULL) {
        int sx = x, sy = y;
        if (!(a.prior_w == a.intr.w && a.prior_h == a.intr.h)) {
            sx = min(x / 2, a.prior_w - 1);
            sy = min(y / 2, a.prior_h - 1);
        }
        const float d = a.prior[static_cast<size_t>(sy) * a.prior_w + sx];
        if (depth_ok(d)) {
            double dd = a.policy_value;
            bool keep = true;
            if (a.policy == FMVS_RANGE_SPACING_MULTIPLE) {
                const double denom = dot3(D3{a.nx, a.ny, a.nz}, unproject_px(a.intr, x, y));
                if (fabs(denom) < 1e-12) {
                    keep = false;
                } else {
                    const double scale = div(-1.0, denom);
                    if (scale <= 0.0) {
                        keep = false;
                    } else {
                        const int i = dev::nearest_index(a.coarser, a.ncoarser, div(double(d), scale));
                        const int j = min(i, a.ncoarser - 2);
                        const double gap = sub(a.coarser[j], a.coarser[j + 1]);
                        dd = mul(mul(a.policy_value, scale), gap);
                    }
                }
            }
            if (keep) {
                const double lo_d = sub(double(d), dd);
                const double hi_d = add(double(d), dd);
                lo = __double2float_rn(a.d_min < lo_d ? lo_d : a.d_min);   // std::max
                hi = __double2float_rn(hi_d < a.d_max ? hi_d : a.d_max);   // std::min
            }
        }
    }
    *lo_f = lo;
    *hi_f = hi;
}

// Plane stacks up to this size are staged in shared memory: the binary
// searches of every pixel read them on their dependency chains.
constexpr int kSmemPlanes = 2048;

__global__ void __launch_bounds__(kRangeThreads) range_rows_kernel(RangeArgs a) {
    using namespace dev;
    using Scan = cub::BlockScan<uint32_t, kRangeThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ uint32_t carry;
    extern __shared__ double s_stack[];  // [nplanes | ncoarser] when both fit
    const int y = blockIdx.x;
    const int w = a.intr.w;
    if (a.nplanes <= kSmemPlanes && (!a.coarser || a.ncoarser <= kSmemPlanes)) {
        for (int i = threadIdx.x; i < a.nplanes; i += kRangeThreads)
            s_stack[i] = a.planes[i];
        if (a.coarser)
            for (int i = threadIdx.x; i < a.ncoarser; i += kRangeThreads)
                s_stack[a.nplanes + i] = a.coarser[i];
        a.planes = s_stack;
        if (a.coarser)
            a.coarser = s_stack + a.nplanes;
    }
    if (threadIdx.x == 0)
        carry = 0;
    __syncthreads();
    for (int x0 = 0; x0 < w; x0 += kRangeThreads) {
        const int x = x0 + threadIdx.x;
        uint32_t first = 0, count = 0;
        if (x < w) {
            float lo, hi;
            pixel_range(a, x, y, &lo, &hi);
            const size_t p = static_cast<size_t>(y) * w + x;
            if (a.lo_out) {
                a.lo_out[p] = lo;
                a.hi_out[p] = hi;
            }
            // pixel_depth_scale (matching.cpp:84-90)
            const double denom = dot3(D3{a.nx, a.ny, a.nz}, unproject_px(a.intr, x, y));
            double scale = 0.0;
            if (!(fabs(denom) < 1e-12)) {
                const double s = div(-1.0, denom);
                scale = s > 0.0 ? s : 0.0;
            }
            const double lod = double(lo), hid = double(hi);
            if (scale > 0.0 && lod <= hid) {
                const int n = a.nplanes;
                // first = #{i : scale*delta_i > hi} (a prefix)
                int l = 0, r = n;
                while (l < r) {
                    const int m = (l + r) >> 1;
                    if (mul(scale, a.planes[m]) > hid)
                        l = m + 1;
                    else
                        r = m;
                }
                const int f = l;
                // s = first i with scale*delta_i < lo (a suffix)
                l = 0;
                r = n;
                while (l < r) {
                    const int m = (l + r) >> 1;
                    if (mul(scale, a.planes[m]) < lod)
                        r = m;
                    else
                        l = m + 1;
                }
                const int last = max(l - 1, f - 1);
                first = static_cast<uint32_t>(f);
                count = static_cast<uint32_t>(max(0, last - f + 1));
            }
        }
        uint32_t excl, agg;
        Scan(scan_tmp).ExclusiveSum(count, excl, agg);
        if (x < w) {
            const size_t p = static_cast<size_t>(y) * w + x;
            a.meta[p] = VolMeta{carry + excl, first | (count << 16)};
        }
        __syncthreads();
        if (threadIdx.x == 0)
            carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0)
        a.row_total[y] = carry;
}

__global__ void __launch_bounds__(1024) scan_rows_kernel(const uint32_t* __restrict__ totals, int h,
                                                        uint64_t* __restrict__ base) {
    using Scan = cub::BlockScan<uint64_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint64_t carry;
    if (threadIdx.x == 0)
        carry = 0;
    __syncthreads();
    for (int y0 = 0; y0 < h; y0 += 1024) {
        const int y = y0 + threadIdx.x;
        const uint64_t v = y < h ? totals[y] : 0;
        uint64_t excl, agg;
        Scan(tmp).ExclusiveSum(v, excl, agg);
        if (y < h)
            base[y] = carry + excl;
        __syncthreads();
        if (threadIdx.x == 0)
            carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0)
        base[h] = carry;
}

}  // namespace

void range_rows(const RangeArgs& a, cudaStream_t s) {
    const size_t smem = (a.nplanes <= kSmemPlanes && (!a.coarser || a.ncoarser <= kSmemPlanes))
                            ? sizeof(double) * (a.nplanes + (a.coarser ? a.ncoarser : 0))
                            : 0;
    // <= 32 KB: within the default dynamic shared-memory limit (no attribute
    // call -- concurrent host threads would race on a per-launch setting)
    range_rows_kernel<<<a.intr.h, kRangeThreads, smem, s>>>(a);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

// agg[0 .. *count) = 0 with contiguous 16-byte stores; the entry count is read
// on the device (row_base[h] of the level), so no host synchronisation.
__global__ void zero_entries_kernel(uint32_t* __restrict__ agg, const uint64_t* __restrict__ count,
                                    bool agg16) {
    const uint64_t n = agg16 ? (*count + 1) / 2 : *count;  // 32-bit words
    const uint64_t n4 = n / 4;
    uint4* a4 = reinterpret_cast<uint4*>(agg);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride)
        a4[i] = make_uint4(0u, 0u, 0u, 0u);
    const uint64_t r = 4 * n4 + blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n)
        agg[r] = 0u;
}

void zero_entries(uint32_t* agg, const uint64_t* count, cudaStream_t s, bool agg16) {
    zero_entries_kernel<<<148 * 4, 512, 0, s>>>(agg, count, agg16);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void scan_rows(const uint32_t* row_total, int h, uint64_t* row_base, cudaStream_t s) {
    scan_rows_kernel<<<1, 1024, 0, s>>>(row_total, h, row_base);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

}  // namespace k
}  // namespace fmvs
