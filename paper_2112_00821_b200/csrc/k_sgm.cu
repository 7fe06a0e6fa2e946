// K6: semi-global path aggregation over the ragged volume (walk_line /
// add_path / aggregate, sgm.cpp:91-239,301-331) for all path directions in
// ONE launch, plus K5 (compute_normal_offsets, sgm.cpp:252-299).
//
// Mapping: one warp per scanline (a line = maximal run along (dx, dy) whose
// first pixel's predecessor lies outside the image, sgm.cpp:213-219). Lanes
// own hypotheses (32 per chunk, any count); the predecessor's path costs live
// in a per-warp shared-memory double buffer because the ragged window of the
// predecessor is offset by prev_first - first - shift. prev_min is one
// __reduce_min_sync (REDUX) per step, the adaptive phi2 comes from a
// host-computed 256-entry LUT, the surface-normal shift from the K5 map, and
// the path-gradient shift from an in-register FP64 scene-point history.
// Path costs are accumulated into the aggregate with integer atomics; integer
// addition commutes, so the result is bit-identical for any schedule (the
// reference's determinism contract, README.md:87-88).
// Roofline: HBM/L2-bound -- per hypothesis and path: 2 B cost read + 4 B
// atomic add; per pixel and path: 8 B meta + 1 B image.
#include "host.hpp"
#include "kernels.hpp"

namespace fmvs {
namespace k {

namespace {

constexpr int kWarps = 4;

__device__ __forceinline__ bool scene_point(const dev::Intr& k, double nx, double ny, double nz,
                                            double dist, int x, int y, dev::D3* out) {
    using namespace dev;  // sgm.cpp:46-58
    const D3 ray = unproject(k, double(x), double(y));
    const double denom = dot3(D3{nx, ny, nz}, ray);
    if (fabs(denom) < 1e-12)
        return false;
    const double t = div(-dist, denom);
    if (t <= 0.0)
        return false;
    *out = scale3(t, ray);
    return true;
}

template <int VARIANT>
__global__ void __launch_bounds__(kWarps * 32) sgm_kernel(SgmArgs a, int total_lines) {
    using namespace dev;
    extern __shared__ uint32_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kWarps + warp;
    if (gw >= total_lines)
        return;
    // Direction d owns the next lines(d) warps (sgm.cpp:231-239 order).
    int rem = gw;
    int d = 0;
    for (; d < a.ndirs; ++d) {
        const int dx = a.dirs[d][0], dy = a.dirs[d][1];
        const int n = (dx != 0 && dy != 0) ? a.h + a.w - 1 : (dy == 0 ? a.h : a.w);
        if (rem < n)
            break;
        rem -= n;
    }
    const int dx = a.dirs[d][0], dy = a.dirs[d][1];
    int x, y;
    if (dy == 0) {
        x = dx > 0 ? 0 : a.w - 1;
        y = rem;
    } else if (dx == 0) {
        x = rem;
        y = dy > 0 ? 0 : a.h - 1;
    } else if (rem < a.h) {
        x = dx > 0 ? 0 : a.w - 1;
        y = rem;
    } else {
        const int k = rem - a.h;  // 0 .. w-2
        x = dx > 0 ? k + 1 : k;
        y = dy > 0 ? 0 : a.h - 1;
    }

    uint32_t* buf_prev;
    uint32_t* buf_cur;
    if (a.scratch) {
        buf_prev = a.scratch + static_cast<size_t>(gw) * 2 * a.pmax;
    } else {
        buf_prev = smem + static_cast<size_t>(warp) * 2 * a.pmax;
    }
    buf_cur = buf_prev + a.pmax;

    // SN: canonical slot and sign of (dx, dy) (sgm.cpp:72-80).
    int slot = 0, sign = 1;
    if (VARIANT == FMVS_SGM_SURFACE_NORMAL) {
        const int cd[4][2] = {{1, 0}, {0, 1}, {1, 1}, {1, -1}};
        for (int c = 0; c < 4; ++c) {
            if (cd[c][0] == dx && cd[c][1] == dy) {
                slot = c;
                sign = 1;
            } else if (cd[c][0] == -dx && cd[c][1] == -dy) {
                slot = c;
                sign = -1;
            }
        }
    }

    bool has_prev = false;
    int prev_first = 0, prev_count = 0, px = 0, py = 0;
    uint32_t prev_min = 0;
    // PG history (sgm.cpp:28-43)
    bool h1 = false, h2 = false;
    D3 p1{0, 0, 0}, p2{0, 0, 0};
    int h1_index = 0;

    while (x >= 0 && y >= 0 && x < a.w && y < a.h) {
        const size_t p = static_cast<size_t>(y) * a.w + x;
        const VolMeta m = a.meta[p];
        const int f = meta_first(m.fc);
        const int c = meta_count(m.fc);
        if (c == 0) {
            has_prev = false;
            h1 = h2 = false;
            x += dx;
            y += dy;
            continue;
        }
        const uint64_t base = a.row_base[y] + m.rel;
        long long phi2 = 0;
        int shift = 0;
        if (has_prev) {
            const int di = abs(int(a.image[p]) - int(a.image[static_cast<size_t>(py) * a.w + px]));
            phi2 = a.phi2_lut[di];
            if (VARIANT == FMVS_SGM_SURFACE_NORMAL && a.offsets) {
                shift = sign * int(a.offsets[4 * p + slot]);
            } else if (VARIANT == FMVS_SGM_PATH_GRADIENT && h1 && h2) {
                const D3 pred = add3(p1, sub3(p1, p2));
                const double delta_pred = -dot3(D3{a.nx, a.ny, a.nz}, pred);
                if (delta_pred > 0.0) {
                    const int pi = dev::nearest_index(a.planes, a.nplanes, delta_pred);
                    shift = min(max(h1_index - pi, -3), 3);
                }
            }
        }
        uint32_t run_min = 0xFFFFFFFFu;
        int run_arg = 0x7FFFFFFF;
        const long long lo = prev_first, hi = prev_first + prev_count;
        for (int i0 = 0; i0 < c; i0 += 32) {
            const int i = i0 + lane;
            if (i < c) {
                const uint32_t s = a.costs[base + i];
                uint32_t v;
                if (!has_prev) {
                    v = s;
                } else {
                    const long long t = static_cast<long long>(f) + i + shift;
                    long long best = static_cast<long long>(prev_min) + phi2;
                    if (t >= lo && t < hi)
                        best = min(best, static_cast<long long>(buf_prev[t - lo]));
                    if (t - 1 >= lo && t - 1 < hi)
                        best = min(best, static_cast<long long>(buf_prev[t - 1 - lo]) + a.phi1);
                    if (t + 1 >= lo && t + 1 < hi)
                        best = min(best, static_cast<long long>(buf_prev[t + 1 - lo]) + a.phi1);
                    v = static_cast<uint32_t>(static_cast<long long>(s) + best -
                                              static_cast<long long>(prev_min));
                }
                buf_cur[i] = v;
                atomicAdd(a.agg + base + i, v);
                if (v < run_min) {
                    run_min = v;
                    run_arg = i;
                }
            }
        }
        prev_min = __reduce_min_sync(0xFFFFFFFFu, run_min);
        if (VARIANT == FMVS_SGM_PATH_GRADIENT) {
            // lowest index attaining the minimum (sgm.cpp:166-174)
            const int arg = __reduce_min_sync(0xFFFFFFFFu, run_min == prev_min ? run_arg : 0x7FFFFFFF);
            D3 pt;
            if (scene_point(a.intr, a.nx, a.ny, a.nz, a.planes[f + arg], x, y, &pt)) {
                h2 = h1;
                p2 = p1;
                h1 = true;
                p1 = pt;
                h1_index = f + arg;
            } else {
                h1 = h2 = false;
            }
        }
        __syncwarp();
        uint32_t* tmp = buf_prev;
        buf_prev = buf_cur;
        buf_cur = tmp;
        has_prev = true;
        prev_first = f;
        prev_count = c;
        px = x;
        py = y;
        x += dx;
        y += dy;
    }
}

// compute_normal_offsets (sgm.cpp:252-299) on the upscaled prior maps.
__global__ void normal_offsets_kernel(OffsetArgs a) {
    using namespace dev;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= a.w || y >= a.h)
        return;
    int sx = x, sy = y;
    if (!(a.prior_w == a.w && a.prior_h == a.h)) {
        sx = min(x / 2, a.prior_w - 1);
        sy = min(y / 2, a.prior_h - 1);
    }
    const size_t sp = static_cast<size_t>(sy) * a.prior_w + sx;
    short4 out = make_short4(0, 0, 0, 0);
    const float nfx = a.prior_normals[3 * sp], nfy = a.prior_normals[3 * sp + 1],
                nfz = a.prior_normals[3 * sp + 2];
    const float depth = a.prior_depth[sp];
    const size_t p = static_cast<size_t>(y) * a.w + x;
    short* o = reinterpret_cast<short*>(&out);
    if (normal_ok(nfx, nfy, nfz) && depth_ok(depth)) {
        const D3 n{double(nfx), double(nfy), double(nfz)};
        const D3 pn{a.nx, a.ny, a.nz};
        const D3 ray = unproject(a.intr, double(x), double(y));
        const double denom0 = dot3(pn, ray);
        if (!(fabs(denom0) < 1e-12 || div(-1.0, denom0) <= 0.0)) {
            const double delta_anchor = mul(double(depth), -denom0);
            const int i0 = dev::nearest_index(a.planes, a.nplanes, delta_anchor);
            const D3 anchor = scale3(div(-a.planes[i0], denom0), ray);
            const int cd[4][2] = {{1, 0}, {0, 1}, {1, 1}, {1, -1}};
            for (int c = 0; c < 4; ++c) {
                const double qx = double(x - cd[c][0]);
                const double qy = double(y - cd[c][1]);
                const D3 ray_q = unproject(a.intr, qx, qy);
                const double denom_t = dot3(n, ray_q);
                if (fabs(denom_t) < 1e-12)
                    continue;
                const double t = div(dot3(n, anchor), denom_t);
                if (t <= 0.0)
                    continue;
                const double delta_q = -dot3(pn, scale3(t, ray_q));
                if (delta_q <= 0.0)
                    continue;
                double df = sub(dev::fractional_index(a.planes, a.nplanes, delta_q), double(i0));
                df = df < -32000.0 ? -32000.0 : (32000.0 < df ? 32000.0 : df);
                o[c] = static_cast<short>(lround(df));
            }
        }
    }
    reinterpret_cast<short4*>(a.out)[p] = out;
}

}  // namespace

void sgm(const SgmArgs& a, cudaStream_t s) {
    int total = 0;
    for (int d = 0; d < a.ndirs; ++d) {
        const int dx = a.dirs[d][0], dy = a.dirs[d][1];
        total += (dx != 0 && dy != 0) ? a.h + a.w - 1 : (dy == 0 ? a.h : a.w);
    }
    if (total == 0)
        return;
    const int blocks = (total + kWarps - 1) / kWarps;
    const size_t smem = a.scratch ? 0 : static_cast<size_t>(kWarps) * 2 * a.pmax * sizeof(uint32_t);
    switch (a.variant) {
        case FMVS_SGM_SURFACE_NORMAL:
            FMVS_CUDA_CHECK(cudaFuncSetAttribute(sgm_kernel<FMVS_SGM_SURFACE_NORMAL>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem)));
            sgm_kernel<FMVS_SGM_SURFACE_NORMAL><<<blocks, kWarps * 32, smem, s>>>(a, total);
            break;
        case FMVS_SGM_PATH_GRADIENT:
            FMVS_CUDA_CHECK(cudaFuncSetAttribute(sgm_kernel<FMVS_SGM_PATH_GRADIENT>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem)));
            sgm_kernel<FMVS_SGM_PATH_GRADIENT><<<blocks, kWarps * 32, smem, s>>>(a, total);
            break;
        default:
            FMVS_CUDA_CHECK(cudaFuncSetAttribute(sgm_kernel<FMVS_SGM_PLANE>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem)));
            sgm_kernel<FMVS_SGM_PLANE><<<blocks, kWarps * 32, smem, s>>>(a, total);
            break;
    }
    FMVS_CUDA_CHECK(cudaGetLastError());
}

// Largest per-warp path buffer that keeps kWarps warps in shared memory.
int sgm_smem_pmax_limit() { return (200 * 1024) / (kWarps * 2 * 4); }

void normal_offsets(const OffsetArgs& a, cudaStream_t s) {
    const dim3 block(32, 8);
    const dim3 grid((a.w + 31) / 32, (a.h + 7) / 8);
    normal_offsets_kernel<<<grid, block, 0, s>>>(a);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

}  // namespace k
}  // namespace fmvs
