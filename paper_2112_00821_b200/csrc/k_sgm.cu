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
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "host.hpp"
#include "kernels.hpp"

namespace fmvs {
namespace k {

namespace {

constexpr int kWarps = 4;

// Lines of one path direction: pixels whose predecessor (x - dx, y - dy) lies
// outside the image (sgm.cpp:213-219), for any step (dx, dy). They form |dx|
// full columns plus |dy| rows of the remaining columns; `rem` enumerates them
// column-major in the first region and row-major in the second, which for
// unit steps is the order of the reference's start scan.
__host__ __device__ __forceinline__ int lines_of_dir(int w, int h, int dx, int dy) {
    const int ax = min(dx < 0 ? -dx : dx, w), ay = min(dy < 0 ? -dy : dy, h);
    return ax * h + (w - ax) * ay;
}

__device__ __forceinline__ void line_start(int w, int h, int dx, int dy, int rem, int* x, int* y) {
    const int ax = min(dx < 0 ? -dx : dx, w), ay = min(dy < 0 ? -dy : dy, h);
    if (rem < ax * h) {
        const int c = rem / h;
        *x = dx > 0 ? c : w - 1 - c;
        *y = rem - c * h;
    } else {
        const int k = rem - ax * h, cols = w - ax;
        const int r = k / cols, c = k - r * cols;
        *x = dx > 0 ? ax + c : c;
        *y = dy > 0 ? r : h - 1 - r;
    }
}

// Direction owning global line index `line` (directions own consecutive
// blocks of lines, in a.dirs order) and the line's first pixel.
__device__ __forceinline__ void locate_line(const SgmArgs& a, int line, int* dx, int* dy, int* x, int* y) {
    int rem = line, d = 0;
    for (; d < a.ndirs - 1; ++d) {
        const int n = lines_of_dir(a.w, a.h, a.dirs[d][0], a.dirs[d][1]);
        if (rem < n)
            break;
        rem -= n;
    }
    *dx = a.dirs[d][0];
    *dy = a.dirs[d][1];
    line_start(a.w, a.h, *dx, *dy, rem, x, y);
}

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

// V is the accumulator type of the recurrence: int64 like the reference, or
// int32 when the host has proven every intermediate fits (sgm() below).
template <int VARIANT, typename V>
__global__ void __launch_bounds__(kWarps * 32) sgm_kernel(SgmArgs a, int total_lines) {
    using namespace dev;
    extern __shared__ uint32_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kWarps + warp;
    if (gw >= total_lines)
        return;
    // Direction d owns the next lines(d) warps (sgm.cpp:231-239 order).
    int dx, dy, x, y;
    locate_line(a, gw, &dx, &dy, &x, &y);

    uint32_t* buf_prev = (a.scratch ? a.scratch + static_cast<size_t>(gw) * 2 * a.pmax
                                    : smem + static_cast<size_t>(warp) * 2 * a.pmax);
    uint32_t* buf_cur = buf_prev + a.pmax;

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
    const bool sn = VARIANT == FMVS_SGM_SURFACE_NORMAL && a.offsets != nullptr;
    const int w = a.w, h = a.h;
    const V phi1 = static_cast<V>(a.phi1);

    // 2-deep software pipeline over the line: per-pixel operands of the
    // current (0) and next (1) pixel are in registers; the first cost chunk
    // of the next pixel and the operands of the one after are loaded while
    // the current pixel's recurrence runs.
    auto inside = [&](int xx, int yy) { return xx >= 0 && yy >= 0 && xx < w && yy < h; };
    VolMeta m0{0u, 0u}, m1{0u, 0u};
    uint64_t rb0 = 0, rb1 = 0;
    int img0 = 0, img1 = 0, off0 = 0, off1 = 0;
    bool v0 = inside(x, y), v1 = inside(x + dx, y + dy);
    if (v0) {
        const size_t p = static_cast<size_t>(y) * w + x;
        m0 = a.meta[p];
        rb0 = a.row_base[y];
        img0 = a.image[p];
        if (sn)
            off0 = a.offsets[4 * p + slot];
    }
    if (v1) {
        const size_t p = static_cast<size_t>(y + dy) * w + x + dx;
        m1 = a.meta[p];
        rb1 = a.row_base[y + dy];
        img1 = a.image[p];
        if (sn)
            off1 = a.offsets[4 * p + slot];
    }
    uint32_t cost0 = 0;
    if (v0 && lane < meta_count(m0.fc))
        cost0 = a.costs[rb0 + m0.rel + lane];

    bool has_prev = false;
    int prev_first = 0, prev_count = 0, img_prev = 0;
    V prev_min = 0;
    // PG history (sgm.cpp:28-43)
    bool h1 = false, h2 = false;
    D3 p1{0, 0, 0}, p2{0, 0, 0};
    int h1_index = 0;

    while (v0) {
        // ---- prefetch: cost chunk 0 of pixel k+1, operands of pixel k+2
        const int x2 = x + 2 * dx, y2 = y + 2 * dy;
        const bool v2 = inside(x2, y2);
        VolMeta m2{0u, 0u};
        uint64_t rb2 = 0;
        int img2 = 0, off2 = 0;
        if (v2) {
            const size_t p = static_cast<size_t>(y2) * w + x2;
            m2 = a.meta[p];
            rb2 = a.row_base[y2];
            img2 = a.image[p];
            if (sn)
                off2 = a.offsets[4 * p + slot];
        }
        uint32_t cost1 = 0;
        if (v1 && lane < meta_count(m1.fc))
            cost1 = a.costs[rb1 + m1.rel + lane];

        // ---- recurrence of pixel k (walk_line, sgm.cpp:97-195)
        const int f = meta_first(m0.fc);
        const int c = meta_count(m0.fc);
        if (c == 0) {
            has_prev = false;
            h1 = h2 = false;
        } else {
            const uint64_t base = rb0 + m0.rel;
            V phi2 = 0;
            int shift = 0;
            if (has_prev) {
                phi2 = static_cast<V>(a.phi2_lut[abs(img0 - img_prev)]);
                if (sn) {
                    shift = sign * off0;
                } else if (VARIANT == FMVS_SGM_PATH_GRADIENT && h1 && h2) {
                    const D3 pred = add3(p1, sub3(p1, p2));
                    const double delta_pred = -dot3(D3{a.nx, a.ny, a.nz}, pred);
                    if (delta_pred > 0.0) {
                        const int pi = dev::nearest_index(a.planes, a.nplanes, delta_pred);
                        shift = min(max(h1_index - pi, -3), 3);
                    }
                }
            }
            const V base_best = prev_min + phi2;
            const int toff = f + shift - prev_first;  // index of hypothesis 0 in prev
            uint32_t run_min = 0xFFFFFFFFu;
            int run_arg = 0x7FFFFFFF;
            for (int i0 = 0; i0 < c; i0 += 32) {
                const int i = i0 + lane;
                if (i < c) {
                    const uint32_t s = i0 == 0 ? cost0 : a.costs[base + i];
                    uint32_t v;
                    if (!has_prev) {
                        v = s;
                    } else {
                        const int t = toff + i;
                        V best = base_best;
                        if (static_cast<unsigned>(t) < static_cast<unsigned>(prev_count))
                            best = min(best, static_cast<V>(buf_prev[t]));
                        if (static_cast<unsigned>(t - 1) < static_cast<unsigned>(prev_count))
                            best = min(best, static_cast<V>(buf_prev[t - 1]) + phi1);
                        if (static_cast<unsigned>(t + 1) < static_cast<unsigned>(prev_count))
                            best = min(best, static_cast<V>(buf_prev[t + 1]) + phi1);
                        v = static_cast<uint32_t>(static_cast<V>(s) + best - prev_min);
                    }
                    buf_cur[i] = v;
                    atomicAdd(a.agg + base + i, v);
                    if (v < run_min) {
                        run_min = v;
                        run_arg = i;
                    }
                }
            }
            const uint32_t nmin = __reduce_min_sync(0xFFFFFFFFu, run_min);
            prev_min = static_cast<V>(nmin);
            if (VARIANT == FMVS_SGM_PATH_GRADIENT) {
                // lowest index attaining the minimum (sgm.cpp:166-174)
                const int arg = __reduce_min_sync(0xFFFFFFFFu, run_min == nmin ? run_arg : 0x7FFFFFFF);
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
            img_prev = img0;
        }
        // ---- rotate the pipeline
        m0 = m1;
        rb0 = rb1;
        img0 = img1;
        off0 = off1;
        cost0 = cost1;
        v0 = v1;
        m1 = m2;
        rb1 = rb2;
        img1 = img2;
        off1 = off2;
        v1 = v2;
        x += dx;
        y += dy;
    }
}

// PlaneStack::nearest_index (geometry.cpp:75-98) with the bracketing index
// found by a local search from `hint` instead of bisection: for a strictly
// decreasing stack the bracket d[lo] >= delta > d[lo + 1] is unique, so the
// result is identical, and along a smooth path it is within a few planes of
// the previous winner.
// Only the rounded index is needed, so the division is skipped where its
// outcome is certain: beyond either end of the stack f <= 0 or f >= n - 1
// (clamped to 0 / n - 1); inside, llround(lo + frac) is lo + 1 exactly when
// frac >= 1/2, decided from 2 * num against den with a 2^-30 relative margin
// (far above the division's and the addition's rounding for lo < 2^11);
// ties within the margin take the reference's exact expression.
__device__ __forceinline__ int nearest_index_from(const double* __restrict__ d, int n, double delta,
                                                  int hint) {
    using namespace dev;
    if (n <= 1 || delta >= d[0])
        return 0;
    if (delta <= d[n - 1])
        return n - 1;
    int lo = min(max(hint, 0), n - 2);
    while (!(d[lo] >= delta))
        --lo;
    while (d[lo + 1] >= delta)
        ++lo;
    const double num = sub(d[lo], delta), den = sub(d[lo], d[lo + 1]);
    const double twice = 2.0 * num;
    if (twice < den * (1.0 - 9.313225746154785e-10))
        return lo;
    if (twice > den * (1.0 + 9.313225746154785e-10))
        return min(lo + 1, n - 1);
    const int i = static_cast<int>(llround(add(double(lo), div(num, den))));
    return i < 0 ? 0 : (i > n - 1 ? n - 1 : i);
}

// PlaneStack::fractional_index (geometry.cpp:75-93) with the bracket found by
// a local search from `hint` (the neighbours' planes lie near the anchor's):
// the bracket d[lo] >= delta > d[lo + 1] of a strictly decreasing stack is
// unique, so the result equals the bisection's.
__device__ __forceinline__ double fractional_index_from(const double* __restrict__ d, int n, double delta,
                                                        int hint) {
    using namespace dev;
    if (n <= 1)
        return 0.0;
    if (delta >= d[0])
        return div(-sub(delta, d[0]), sub(d[0], d[1]));
    if (delta <= d[n - 1])
        return add(double(n - 1), div(sub(d[n - 1], delta), sub(d[n - 2], d[n - 1])));
    int lo = min(max(hint, 0), n - 2);
    while (!(d[lo] >= delta))
        --lo;
    while (d[lo + 1] >= delta)
        ++lo;
    return add(double(lo), div(sub(d[lo], delta), sub(d[lo], d[lo + 1])));
}

// Minimum over the G-lane group of the calling lane (G a power of two): a
// full-warp REDUX for G = 32, an xor butterfly otherwise (a group-masked
// REDUX with per-group masks serialises into one pass per group).
template <int G>
__device__ __forceinline__ uint32_t group_min(uint32_t v) {
    if (G == 32)
        return __reduce_min_sync(0xFFFFFFFFu, v);
#pragma unroll
    for (int o = 1; o < G; o <<= 1)
        v = min(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    return v;
}

// Operands of one pixel of a scanline, staged in registers ahead of its step.
template <int K, typename V>
struct LinePx {
    // stage 1: raw loads only, each landing in its final register as loaded
    // (no conversion or arithmetic on a value in flight: any instruction that
    // touches it, even a zero-extension, waits for the load)
    uint64_t rb;     // row base of the pixel's row
    dev::VolMeta m;  // {offset in row, first | count << 16}
    uint32_t img4;   // 32-bit word (or zero-extended byte) holding the intensity
    uint32_t off2;   // aligned 32-bit word holding the SN shift (int16)
    int img_sh;      // bit offset of the intensity in img4
    bool v;          // inside the image
    // stage 2
    uint64_t base;   // entry index of hypothesis 0
    int img;         // reference intensity
    V phi2;          // phi2 of the transition from the previous pixel
    uint32_t s[K];   // costs of the first pass
};

#ifndef FMVS_SGM_SLOTS
#define FMVS_SGM_SLOTS 8
#endif
#ifndef FMVS_SGM_GAP
#define FMVS_SGM_GAP 3
#endif
constexpr int kSgmSlots = FMVS_SGM_SLOTS;  // register pipeline depth (pixels in flight per line)
constexpr int kGap = FMVS_SGM_GAP;         // steps between a pixel's meta load and its cost loads
constexpr int kSent = 3;      // sentinel slots on each side of a path buffer
constexpr uint32_t kSentinel = 0x3FFFFFFFu;

// Register-blocked variant (Plane / SurfaceNormal): G lanes per scanline and
// 32/G scanlines per warp; lane gl owns the K hypotheses i = gl + G*k of a
// pass of G*K (pixels wider than a pass loop over passes). At the refined
// levels a pixel has ~12 hypotheses, so G=4, K=4 covers it in one pass with 8
// scanlines per warp.
//
// The recurrence is sequential along a line, so the kernel is bound by the
// latency of one step. The operands are therefore staged through a
// kSgmSlots-deep register pipeline, unrolled so that no slot is ever copied (a
// register copy would wait for its pending load): at the step of pixel k the
// meta / image / SN shift of pixel k+7 are loaded, the first-pass costs of
// pixel k+4 (whose meta was requested kGap = 3 steps earlier) are loaded and
// its phi2 is looked up, and pixel k is computed from operands requested 4-7
// steps earlier.
//
// Path buffers: a per-line shared-memory double buffer (line stride padded so
// the 32/G lines of a warp start in distinct banks); pixels wider than `caps`
// hypotheses spill to a per-line global buffer. In the int32 recurrence (SENT)
// every buffer carries kSent sentinel slots on both sides, so the ragged
// predecessor window prev[t-1..t+1] needs no bounds tests: t is clamped into
// [-2, prev_count + 1] and out-of-range slots read kSentinel, which never
// beats prev_min + phi2 (all path values stay below 2^30 when the host picks
// the int32 path).
template <int VARIANT, typename V, int G, int K>
__global__ void __launch_bounds__(kWarps * 32) sgm_lanes_kernel(SgmArgs a, int total_lines,
                                                                int caps, int stride) {
    using namespace dev;
    constexpr bool SENT = sizeof(V) == 4;
    constexpr int LPW = 32 / G;
    constexpr int PASS = G * K;
    // wide passes (dense coarsest levels, K = 8) keep fewer pixels in flight:
    // each step is longer, and the slots' cost registers scale with K
    constexpr int S = K >= 8 ? 4 : kSgmSlots;
    constexpr int GAP = K >= 8 ? 1 : kGap;
    extern __shared__ uint32_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / G, gl = lane % G;
    const int line = (blockIdx.x * kWarps + warp) * LPW + grp;
    const int w = a.w, h = a.h;

    int dx = 1, dy = 0, x = -1, y = -1;
    if (line < total_lines)
        locate_line(a, line, &dx, &dy, &x, &y);
    // buffer layout (both smem and global): [kSent sentinels][caps or pmax][kSent]
    uint32_t* sA = smem + static_cast<size_t>(warp * LPW + grp) * stride + kSent;
    uint32_t* sB = sA + caps + 2 * kSent;
    const size_t gstride = static_cast<size_t>(a.pmax) + 2 * kSent;
    uint32_t* gA = (a.scratch && line < total_lines) ? a.scratch + static_cast<size_t>(line) * 2 * gstride + kSent
                                                     : nullptr;
    uint32_t* gB = gA ? gA + gstride : nullptr;
    if (SENT && gl < kSent) {
        sA[-kSent + gl] = kSentinel;
        sB[-kSent + gl] = kSentinel;
        if (gA) {
            gA[-kSent + gl] = kSentinel;
            gB[-kSent + gl] = kSentinel;
        }
    }
    __syncwarp();  // sentinels visible to the group before its first window read

    // SN: canonical slot of +-(dx, dy) among (1,0), (0,1), (1,1), (1,-1) and the
    // sign of the direction (sgm.cpp:72-87), in closed form
    const int slot = dy == 0 ? 0 : (dx == 0 ? 1 : (dx == dy ? 2 : 3));
    const int sign = (dy == 0 || dx == 0) ? dx + dy : dx;
    const bool sn = VARIANT == FMVS_SGM_SURFACE_NORMAL && a.offsets != nullptr;
    const V phi1 = static_cast<V>(a.phi1);
    auto inside = [&](int xx, int yy) { return xx >= 0 && yy >= 0 && xx < w && yy < h; };

    using Px = LinePx<K, V>;
    Px P[S];
    // stage 1: meta, row base, image word, SN shift word (raw)
    const uintptr_t img_lo = reinterpret_cast<uintptr_t>(a.image);
    const uintptr_t img_hi = img_lo + static_cast<uintptr_t>(w) * h;
    const int off_sh = (slot & 1) * 16;
    auto load_meta = [&](Px& q, int xx, int yy, bool valid) {
        q.v = valid;
        q.m = dev::VolMeta{0u, 0u};
        q.rb = 0;
        q.img4 = 0;
        q.off2 = 0;
        q.img_sh = 0;
        if (valid) {
            const size_t p = static_cast<size_t>(yy) * w + xx;
            q.m = a.meta[p];
            q.rb = a.row_base[yy];
            // aligned 32-bit word holding the byte when it lies inside the
            // image (a byte load otherwise); either lands in the slot register
            // with no conversion
            const uintptr_t ia = reinterpret_cast<uintptr_t>(a.image + p);
            const uintptr_t wa = ia & ~uintptr_t(3);
            if (wa >= img_lo && wa + 4 <= img_hi) {
                q.img4 = __ldg(reinterpret_cast<const uint32_t*>(wa));
                q.img_sh = static_cast<int>(ia - wa) * 8;
            } else {
                q.img4 = __ldg(a.image + p);
            }
            if (sn)
                q.off2 = __ldg(reinterpret_cast<const uint32_t*>(a.offsets + 4 * p) + (slot >> 1));
        }
    };
    // stage 2: entry base, intensity, first-pass costs, phi2 of the
    // transition from the previous pixel
    auto load_costs = [&](Px& q, const Px& qprev) {
        const int c = meta_count(q.m.fc);
        q.base = q.rb + q.m.rel;
        q.img = static_cast<int>((q.img4 >> q.img_sh) & 0xFFu);
        const uint16_t* cp = a.costs + q.base;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int i = gl + G * k;
            q.s[k] = i < c ? cp[i] : 0u;
        }
        q.phi2 = (q.v && qprev.v) ? static_cast<V>(a.phi2_lut[abs(q.img - qprev.img)]) : V(0);
    };

    // prologue: pixels 0..S-2 through stage 1, pixels 0..S-4 through stage 2
    {
        bool valid = inside(x, y);
#pragma unroll
        for (int j = 0; j < S - 1; ++j) {
            load_meta(P[j], x + j * dx, y + j * dy, valid);
            valid = valid && inside(x + (j + 1) * dx, y + (j + 1) * dy);
        }
        P[S - 1].v = false;
        P[S - 1].img = 0;
        P[S - 1].img4 = 0;
        P[S - 1].img_sh = 0;
#pragma unroll
        for (int j = 0; j < S - 1 - GAP; ++j)
            load_costs(P[j], P[(j + S - 1) % S]);
    }

    bool has_prev = false;
    int prev_first = 0, prev_count = 0;
    V prev_min = 0;
    const uint32_t* prev = sA;
    // PG history of the line (sgm.cpp:28-43): the two previous winners' scene
    // points; every lane of the group carries an identical copy
    constexpr bool PG = VARIANT == FMVS_SGM_PATH_GRADIENT;
    bool h1 = false, h2 = false;
    D3 p1{0, 0, 0}, p2{0, 0, 0};
    int h1_index = 0;

    for (;;) {
#pragma unroll
        for (int u = 0; u < S; ++u) {
            Px& cur_px = P[u];
            if (!__any_sync(0xFFFFFFFFu, cur_px.v))
                goto done;
            // stage 1 for pixel k+S-1, stage 2 for pixel k+S-3
            {
                Px& pn = P[(u + S - 1) % S];
                const Px& pl = P[(u + S - 2) % S];
                load_meta(pn, x + (S - 1) * dx, y + (S - 1) * dy,
                          pl.v && inside(x + (S - 1) * dx, y + (S - 1) * dy));
                load_costs(P[(u + S - 1 - GAP) % S], P[(u + S - 2 - GAP) % S]);
            }
            // recurrence of pixel k (walk_line, sgm.cpp:97-195)
            const int f = meta_first(cur_px.m.fc);
            const int c = cur_px.v ? meta_count(cur_px.m.fc) : 0;
            uint32_t run_min = 0xFFFFFFFFu;
            int run_arg = 0x7FFFFFFF;
            uint32_t* cur = nullptr;
            if (c > 0) {
                cur = c <= caps ? (prev == sA ? sB : sA) : (prev == gA ? gB : gA);
                const V phi2 = has_prev ? cur_px.phi2 : V(0);
                int shift =
                    (has_prev && sn) ? sign * static_cast<int>(static_cast<int16_t>(cur_px.off2 >> off_sh)) : 0;
                if (PG && has_prev && h1 && h2) {  // sgm.cpp:131-140
                    const D3 pred = add3(p1, sub3(p1, p2));
                    const double delta_pred = -dot3(D3{a.nx, a.ny, a.nz}, pred);
                    if (delta_pred > 0.0) {
                        const int pi = nearest_index_from(a.planes, a.nplanes, delta_pred, h1_index);
                        shift = min(max(h1_index - pi, -3), 3);
                    }
                }
                const V base_best = prev_min + phi2;
                const int toff = f + shift - prev_first;
                const uint16_t* cp = a.costs + cur_px.base;
                uint32_t* ap = a.agg + cur_px.base;
                if (SENT) {
                    // branch-free: the clamped window reads sentinels (or stale
                    // slots) for inactive lanes, whose result is discarded; no
                    // previous pixel adds nothing. The first pass (the only one
                    // at refined levels) is straight-line code on the
                    // prefetched costs; further passes load theirs.
                    auto pass = [&](int i0, auto first) {
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            const int i = i0 + gl + G * k;
                            const bool act = i < c;
                            uint32_t sc;
                            if constexpr (decltype(first)::value)
                                sc = cur_px.s[k];
                            else
                                sc = act ? cp[i] : 0u;
                            const int t = min(max(toff + i, -2), prev_count + 1);
                            const V b3 = min(static_cast<V>(prev[t - 1]), static_cast<V>(prev[t + 1])) + phi1;
                            const V best = min(min(base_best, static_cast<V>(prev[t])), b3);
                            const uint32_t v = sc + (has_prev ? static_cast<uint32_t>(best - prev_min) : 0u);
                            if (act) {
                                cur[i] = v;
                                atomicAdd(ap + i, v);
                            }
                            if (PG) {
                                if (act && v < run_min) {  // lanes scan ascending i
                                    run_min = v;
                                    run_arg = i;
                                }
                            } else {
                                run_min = min(run_min, act ? v : 0xFFFFFFFFu);
                            }
                        }
                    };
                    pass(0, std::true_type{});
                    for (int i0 = PASS; i0 < c; i0 += PASS)
                        pass(i0, std::false_type{});
                } else {
                    for (int i0 = 0; i0 < c; i0 += PASS) {
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            const int i = i0 + gl + G * k;
                            if (i >= c)
                                continue;
                            const uint32_t sc = i0 == 0 ? cur_px.s[k] : cp[i];
                            uint32_t v;
                            if (!has_prev) {
                                v = sc;
                            } else {
                                const int t = toff + i;
                                V best = base_best;
                                if (static_cast<unsigned>(t) < static_cast<unsigned>(prev_count))
                                    best = min(best, static_cast<V>(prev[t]));
                                if (static_cast<unsigned>(t - 1) < static_cast<unsigned>(prev_count))
                                    best = min(best, static_cast<V>(prev[t - 1]) + phi1);
                                if (static_cast<unsigned>(t + 1) < static_cast<unsigned>(prev_count))
                                    best = min(best, static_cast<V>(prev[t + 1]) + phi1);
                                v = static_cast<uint32_t>(static_cast<V>(sc) + best - prev_min);
                            }
                            cur[i] = v;
                            atomicAdd(ap + i, v);
                            if (v < run_min) {
                                run_min = v;
                                run_arg = i;
                            }
                        }
                    }
                }
                if (SENT && gl < kSent)
                    cur[c + gl] = kSentinel;
            }
            const uint32_t nmin = group_min<G>(run_min);
            if (PG) {
                // lowest index attaining the minimum (sgm.cpp:166-174), then
                // its scene point (sgm.cpp:176-185, scene_point :46-58)
                const int arg = static_cast<int>(
                    group_min<G>(run_min == nmin ? static_cast<uint32_t>(run_arg) : 0x7FFFFFFFu));
                if (c > 0) {
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
                } else {
                    h1 = h2 = false;  // empty pixel resets the path (sgm.cpp:101-106)
                }
            }
            __syncwarp();
            if (c > 0) {
                prev_min = static_cast<V>(nmin);
                prev = cur;
                has_prev = true;
                prev_first = f;
                prev_count = c;
            } else {
                has_prev = false;
            }
            x += dx;
            y += dy;
        }
    }
done:
    return;
}

// ---- line kernel: Plane / SurfaceNormal, unit directions, int32 ------------
//
// Same recurrence and mapping as sgm_lanes_kernel (G lanes per scanline, K
// hypotheses per lane and pass), restructured so that a step costs few
// instructions:
//  * every per-pixel operand of a step comes from ONE 48-byte record built
//    per level by sgm_prep_kernel: a 16-byte head (32-bit entry index; first
//    | count << 11 | intensity << 23; the four SN shifts) and, for pixels of
//    <= kEmbed hypotheses, a copy of the pixel's u16 costs laid out per lane
//    (slot 4*gl + k holds hypothesis gl + 4k), so a step issues one head load
//    and one 8-byte cost load per lane, both addressed by the pixel index
//    alone: no load waits on another (instead of meta + row base + image +
//    SN loads, then cost loads addressed by the meta); records past the end
//    of a line read a zero dummy record;
//  * the line's length is known at its start (no per-step inside tests, the
//    warp runs max-length steps);
//  * the path buffers of a line live in ONE address space for the whole line,
//    chosen at its start: shared memory, or the global scratch when any pixel
//    of the line is wider than the shared capacity (flagged by the prep
//    kernel per row / column / diagonal / anti-diagonal); the double buffer
//    alternates on every step, so with an even pipeline depth its parity is
//    static in the unrolled step loop;
//  * a pixel without a predecessor reads only the three left sentinels (its
//    window offset is pushed far left), so no has_prev selects in the
//    hypothesis loop; the phi2 LUT lives in shared memory.
// Records hold 32-bit entry indices and <= kRecPlanes planes (host-checked;
// other volumes take the general kernel).
constexpr int kRecPlanes = 2048;
constexpr int kRecWords = 12;  // 48-byte record: head + 16 embedded u16 costs
constexpr int kEmbed = 16;     // pixels with more hypotheses keep only the head

__device__ __forceinline__ int rec_first(uint32_t pk) { return static_cast<int>(pk & 0x7FFu); }
__device__ __forceinline__ int rec_count(uint32_t pk) { return static_cast<int>((pk >> 11) & 0xFFFu); }
__device__ __forceinline__ int rec_img(uint32_t pk) { return static_cast<int>(pk >> 23); }

// wide-line flags: one word per row, column, diagonal (x - y) and
// anti-diagonal (x + y)
struct LineFlags {
    uint32_t* row;
    uint32_t* col;
    uint32_t* diag;
    uint32_t* anti;
};
__host__ __device__ inline LineFlags line_flags(uint32_t* base, int w, int h) {
    return {base, base + h, base + h + w, base + h + w + (w + h - 1)};
}
__host__ __device__ inline size_t line_flag_words(int w, int h) {
    return static_cast<size_t>(h) + w + 2 * (static_cast<size_t>(w) + h - 1);
}

template <typename F, int... I>
__device__ __forceinline__ void static_for_impl(F& f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
}
// f(integral_constant<int, 0>) ... f(integral_constant<int, N - 1>)
template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// Aggregate RED of (p ? v : 0) at a byte offset, UNCONDITIONAL: straight-line
// code (a predicated or guarded RED compiles to a branch per hypothesis). An
// inactive lane adds 0 to an entry of a later pixel, or to the kAggSlack
// entries every aggregate allocation carries past the volume's last entry.
template <int OFF>
__device__ __forceinline__ void red_add(uint32_t* agg, bool p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0+%1], %2;" : : "l"(agg), "n"(OFF), "r"(p ? v : 0u));
}

// embed: 0 head only (16-byte records), 1 + u16 costs (48 bytes: slot 4*gl + k
// = hypothesis gl + 4k), 2 + 10-bit costs (32 bytes: lane gl's word holds
// hypotheses gl + 4k, k < 3, at bits 10k); see LinePipe.
__global__ void sgm_prep_kernel(SgmArgs a, uint4* rec, LineFlags fl, int caps, int embed) {
    const int n = a.w * a.h;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > n)
        return;
    const int rs = embed == 0 ? 1 : (embed == 1 ? 3 : 2);
    uint4* r = rec + static_cast<size_t>(rs) * p;
    if (p == n) {  // the dummy record read past the end of a line
        for (int k = 0; k < rs; ++k)
            r[k] = make_uint4(0u, 0u, 0u, 0u);
        return;
    }
    const int y = p / a.w, x = p - y * a.w;
    const dev::VolMeta m = a.meta[p];
    const int c = dev::meta_count(m.fc);
    const uint64_t base = a.row_base[y] + m.rel;
    uint4 h;
    h.x = static_cast<uint32_t>(base);
    h.y = (c > 0 ? static_cast<uint32_t>(dev::meta_first(m.fc)) : 0u) | static_cast<uint32_t>(c) << 11 |
          static_cast<uint32_t>(a.image[p]) << 23;
    if (a.offsets) {
        const uint2 o = reinterpret_cast<const uint2*>(a.offsets)[p];
        h.z = o.x;
        h.w = o.y;
    } else {
        h.z = h.w = 0u;
    }
    r[0] = h;
    if (embed == 1) {
        uint32_t e[8];
#pragma unroll
        for (int sl = 0; sl < 16; sl += 2) {
            uint32_t v2 = 0u;
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                const int slot = sl + h2;
                const int i = (slot >> 2) + 4 * (slot & 3);
                if (c <= kEmbed && i < c)
                    v2 |= static_cast<uint32_t>(a.costs[base + i]) << (16 * h2);
            }
            e[sl >> 1] = v2;
        }
        r[1] = make_uint4(e[0], e[1], e[2], e[3]);
        r[2] = make_uint4(e[4], e[5], e[6], e[7]);
    } else if (embed == 2) {
        uint32_t e[4];
#pragma unroll
        for (int gl = 0; gl < 4; ++gl) {
            uint32_t wd = 0u;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int i = gl + 4 * k;
                if (c <= 12 && i < c)
                    wd |= (static_cast<uint32_t>(a.costs[base + i]) & 0x3FFu) << (10 * k);
            }
            e[gl] = wd;
        }
        r[1] = make_uint4(e[0], e[1], e[2], e[3]);
    }
    if (c > caps) {
        atomicOr(fl.row + y, 1u);
        atomicOr(fl.col + x, 1u);
        atomicOr(fl.diag + (x - y + a.h - 1), 1u);
        atomicOr(fl.anti + (x + y), 1u);
    }
}

// Per-line constants of the line kernel.
struct LineCtx {
    const uint4* __restrict__ rec;
    const int* lut;  // phi2 LUT (shared memory)
    int gl;          // lane within the line's group
    int n;           // pixels on the line
    int steps;       // steps the warp runs (>= n)
    int q;           // pixel index of the line's first pixel
    int dp;          // pixel-index step along the line
    int dummy;       // index of the zero record
    int sign, off_sh;
    bool off_hi;
    int x0, y0, dx, dy;  // first pixel and step of the line (PG scene points)
    const double* planes;  // PG: the plane stack (shared-memory copy)
    int rs;                // record stride in 16-byte units (1: head only, 3: + u16 costs, 2: + 10-bit costs)
};

// Operand pipeline of the line kernel: records of pixels j+1..j+S-1 and the
// costs / phi2 of pixels j+1..j+S-1-GAP in registers at the step of pixel j.
// EMB: the costs come with the record (embedded copy, G = 4, K <= 4) and phi2
// is looked up at use; otherwise they are loaded GAP steps after the record.
// EMB: 0 costs from the volume (loaded GAP steps after the record), 1 u16
// costs embedded in the record, 2 10-bit costs packed one word per lane (K <=
// 3, every cost < 1024); with 1 and 2 phi2 is looked up a step ahead.
template <bool SN, int G, int K, int S, int GAP, int EMB>
struct LinePipe {
    static_assert(!EMB || (G == 4 && K <= 4), "embedded costs hold 4 slots for 4 lanes");
    static_assert(EMB != 2 || K <= 3, "three 10-bit costs per lane word");
    uint4 R[S];
    uint2 E[EMB == 1 ? S : 1];
    uint32_t E10[EMB == 2 ? S : 1];
    uint32_t C[EMB ? 1 : S][K];
    int PH[EMB ? 1 : S];
    int q, jn;

    __device__ __forceinline__ void load_rec(const LineCtx& lc, int si) {
        const int idx = jn < lc.n ? q : lc.dummy;
        const uint4* r = lc.rec + lc.rs * idx;
        if (SN) {
            R[si] = __ldg(r);
        } else {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(r));
            R[si].x = v.x;
            R[si].y = v.y;
            R[si].z = R[si].w = 0u;
        }
        if constexpr (EMB == 1)
            E[si] = __ldg(reinterpret_cast<const uint2*>(r + 1) + lc.gl);
        else if constexpr (EMB == 2)
            E10[si] = __ldg(reinterpret_cast<const uint32_t*>(r + 1) + lc.gl);
        q += lc.dp;
        ++jn;
    }
    // first-pass cost k of the pixel in slot u
    __device__ __forceinline__ uint32_t cost(int u, int k) const {
        if constexpr (EMB == 1)
            return ((k < 2 ? E[u].x : E[u].y) >> (16 * (k & 1))) & 0xFFFFu;
        else if constexpr (EMB == 2)
            return (E10[u] >> (10 * k)) & 0x3FFu;
        else
            return C[u][k];
    }
    __device__ __forceinline__ void load_costs(const SgmArgs& a, const LineCtx& lc, int si, int sp) {
        if constexpr (EMB)
            return;
        const uint32_t pk = R[si].y;
        const int c = rec_count(pk);
        const uint16_t* cp = a.costs + (R[si].x + lc.gl);
#pragma unroll
        for (int k = 0; k < K; ++k)
            C[si][k] = lc.gl + G * k < c ? cp[G * k] : 0u;
        PH[si] = lc.lut[abs(rec_img(pk) - rec_img(R[sp].y))];
    }
    // prologue: records of pixels 0..S-2, costs of pixels 0..S-2-GAP
    __device__ __forceinline__ void start(const SgmArgs& a, const LineCtx& lc) {
        q = lc.q;
        jn = 0;
#pragma unroll
        for (int j = 0; j < S - 1; ++j)
            load_rec(lc, j);
        R[S - 1] = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int j = 0; j < S - 1 - GAP; ++j)
            load_costs(a, lc, j, (j + S - 1) % S);
    }
    // at the step in slot u: record of pixel j+S-1 (into the slot of pixel
    // j-1), costs of pixel j+S-1-GAP (its record arrived GAP steps ago)
    __device__ __forceinline__ void advance(const SgmArgs& a, const LineCtx& lc, int u) {
        load_rec(lc, (u + S - 1) % S);
        load_costs(a, lc, (u + S - 1 - GAP) % S, (u + S - 2 - GAP) % S);
    }
    __device__ __forceinline__ int shift(const LineCtx& lc, int u) const {
        const uint32_t wd = lc.off_hi ? R[u].w : R[u].z;
        return lc.sign * static_cast<int>(static_cast<int16_t>(wd >> lc.off_sh));
    }
};

// Steps of the lines of a warp: any number of passes per pixel (pixels wider
// than G*K hypotheses loop), each line's double buffer in shared memory or,
// when the line is wide, in its global scratch (SHARED: no line of the warp
// is wide, so the buffers are shared-memory typed). Each step is its own
// basic block (the `c > 0` branch), which keeps the compiler from sinking the
// pipelined record and cost loads towards their uses (measured: branch-free
// step bodies, with the predecessor window loaded a step early, ran 1.8x
// slower at level 0, with the same loads staged through shared memory by
// cp.async too).
template <bool SN, int G, int K, int S, int GAP, bool SHARED, int EMB, bool AGG16, bool PG>
__device__ __forceinline__ void line_steps(const SgmArgs& a, const LineCtx& lc, uint32_t* bufA,
                                          uint32_t* bufB) {
    constexpr int PASS = G * K;
    const int gl = lc.gl;
    const int phi1 = static_cast<int>(a.phi1);
    LinePipe<SN, G, K, S, GAP, EMB> P;
    P.start(a, lc);
    int prev_count = 0, prev_min = 0, ph = 0, toff = -0x40000000;
    bool has_prev = false;
    // PG: minimum-cost history of the line (sgm.cpp:28-43), the same in every
    // lane of the group; the pixel's coordinates for its scene point
    bool h1 = false, h2 = false;
    dev::D3 p1{0.0, 0.0, 0.0}, p2{0.0, 0.0, 0.0};
    int h1_index = 0;
    int px = lc.x0, py = lc.y0;
    // first-pass predecessor window of the current pixel (prev[t-1], prev[t],
    // prev[t+1] per slot), loaded at the end of the previous step so the
    // loads overlap the group-minimum shuffles
    int W0[K], W1[K], W2[K];
#pragma unroll
    for (int k = 0; k < K; ++k)
        W0[k] = W1[k] = W2[k] = static_cast<int>(kSentinel);
    for (int j0 = 0; j0 < lc.steps; j0 += S) {
#pragma unroll
        for (int u = 0; u < S; ++u) {
            P.advance(a, lc, u);
            uint32_t* cur = (u & 1) ? bufA : bufB;
            const uint32_t* prev = (u & 1) ? bufB : bufA;
            const uint32_t pk = P.R[u].y;
            const int c = rec_count(pk), f = rec_first(pk);
            uint32_t run_min = 0xFFFFFFFFu;
            int run_arg = 0x7FFFFFFF;  // PG: lowest index attaining run_min (lanes scan i upwards)
            // PG: the pixel's viewing ray and its plane-normal dot (scene_point,
            // sgm.cpp:46-58), computed before the recurrence so the divisions
            // stay off the winner -> shift dependency chain
            dev::D3 ray{0.0, 0.0, 1.0};
            double denom = 0.0;
            if constexpr (PG) {
                // the divisions, not the table: a table load here sits on
                // the step's dependency chain (measured slower)
                ray = dev::unproject(a.intr, double(px), double(py));
                denom = dev::dot3(dev::D3{a.nx, a.ny, a.nz}, ray);
            }
            if (c > 0) {
                const int pm = has_prev ? prev_min : 0;
                const int bp = has_prev ? prev_min + (EMB ? ph : P.PH[u]) : 0;
                const int tmax = prev_count + 1;
                const uint32_t ib = P.R[u].x + gl;
                auto pass = [&](int i0, const uint32_t* sc, bool first) {
                    // AGG16: entry e is u16 e of the aggregate (two per word);
                    // the lanes' entries of a pass share e's parity (G even)
                    const uint32_t e0 = ib + i0;
                    uint32_t* ap = AGG16 ? a.agg + (e0 >> 1) : a.agg + e0;
                    const int sh = AGG16 ? static_cast<int>(e0 & 1u) * 16 : 0;
                    uint32_t* cp = cur + (gl + i0);
                    static_for<K>([&](auto kc) {
                        constexpr int k = decltype(kc)::value;
                        const int i = i0 + gl + G * k;
                        int w0, w1, w2;
                        if (first) {
                            w0 = W0[k];
                            w1 = W1[k];
                            w2 = W2[k];
                        } else {
                            const int t = min(max(toff + i, -2), tmax);
                            w0 = static_cast<int>(prev[t - 1]);
                            w1 = static_cast<int>(prev[t]);
                            w2 = static_cast<int>(prev[t + 1]);
                        }
                        const int best = min(min(bp, w1), min(w0, w2) + phi1);
                        const uint32_t v = sc[k] + static_cast<uint32_t>(best - pm);
                        if (i < c)
                            cp[G * k] = v;
                        if constexpr (AGG16)
                            red_add<2 * G * k>(ap, i < c, v << sh);
                        else
                            red_add<4 * G * k>(ap, i < c, v);
                        if constexpr (PG) {
                            if (i < c && v < run_min) {
                                run_min = v;
                                run_arg = i;
                            }
                        } else {
                            run_min = min(run_min, i < c ? v : 0xFFFFFFFFu);
                        }
                    });
                };
                uint32_t sc0[K];
#pragma unroll
                for (int k = 0; k < K; ++k)
                    sc0[k] = P.cost(u, k);
                pass(0, sc0, true);
                for (int i0 = PASS; i0 < c; i0 += PASS) {
                    const uint16_t* cp = a.costs + (ib + i0);
                    uint32_t sc[K];
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        sc[k] = i0 + gl + G * k < c ? cp[G * k] : 0u;
                    pass(i0, sc, false);
                }
                if (gl < kSent)
                    cur[c + gl] = kSentinel;
            }
            __syncwarp();
            int pg_shift = 0;
            if constexpr (PG) {
                // winner of this pixel (sgm.cpp:166-174) and its scene point
                // (:176-185), then the predicted shift of the next pixel
                // (:131-140, nearest_index by a local bracket search)
                const uint32_t nmin_pg = group_min<G>(run_min);
                const int arg = static_cast<int>(
                    group_min<G>(run_min == nmin_pg ? static_cast<uint32_t>(run_arg) : 0x7FFFFFFFu));
                if (c > 0) {
                    const double t = fabs(denom) < 1e-12 ? 0.0 : dev::div(-lc.planes[f + arg], denom);
                    if (t > 0.0) {
                        h2 = h1;
                        p2 = p1;
                        h1 = true;
                        p1 = dev::scale3(t, ray);
                        h1_index = f + arg;
                    } else {
                        h1 = h2 = false;
                    }
                    if (h1 && h2) {
                        const dev::D3 pred = dev::add3(p1, dev::sub3(p1, p2));
                        const double delta_pred = -dev::dot3(dev::D3{a.nx, a.ny, a.nz}, pred);
                        if (delta_pred > 0.0) {
                            const int pi = nearest_index_from(lc.planes, a.nplanes, delta_pred, h1_index);
                            pg_shift = min(max(h1_index - pi, -3), 3);
                        }
                    }
                } else {
                    h1 = h2 = false;  // an empty pixel resets the path (sgm.cpp:101-106)
                }
                px += lc.dx;
                py += lc.dy;
            }
            // predecessor window of pixel j+1 in this pixel's buffer (an empty
            // pixel leaves only the permanent left sentinels in reach)
            {
                const int u1 = (u + 1) % S;
                const int shift = SN ? P.shift(lc, u1) : pg_shift;
                toff = c > 0 ? rec_first(P.R[u1].y) + shift - f : -0x40000000;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int t = min(max(toff + gl + G * k, -2), c + 1);
                    W0[k] = static_cast<int>(cur[t - 1]);
                    W1[k] = static_cast<int>(cur[t]);
                    W2[k] = static_cast<int>(cur[t + 1]);
                }
            }
            const uint32_t nmin = group_min<G>(run_min);
            if (c > 0) {
                prev_min = static_cast<int>(nmin);
                prev_count = c;
            }
            has_prev = c > 0;
            if (EMB)  // phi2 of the transition into the next pixel, a step ahead
                ph = lc.lut[abs(rec_img(P.R[(u + 1) % S].y) - rec_img(pk))];
        }
    }
}

template <bool SN, int G, int K, int S, int GAP, int EMB, bool AGG16, bool PG>
__global__ void __launch_bounds__(kWarps * 32) sgm_line_kernel(SgmArgs a, const uint4* __restrict__ rec,
                                                               LineFlags fl, int total_lines, int stride) {
    constexpr int LPW = 32 / G;
    constexpr int PASS = G * K;
    static_assert(S % 2 == 0, "static double-buffer parity needs an even pipeline depth");
    extern __shared__ uint32_t smem[];
    int* lut = reinterpret_cast<int*>(smem);
    for (int i = threadIdx.x; i < 256; i += kWarps * 32)
        lut[i] = static_cast<int>(a.phi2_lut[i]);
    // PG: the plane stack after the path buffers (its bracket searches and
    // scene points sit on the step's dependency chain)
    double* s_planes = reinterpret_cast<double*>(smem + ((256 + kWarps * LPW * stride + 1) & ~1));
    if (PG)
        for (int i = threadIdx.x; i < a.nplanes; i += kWarps * 32)
            s_planes[i] = a.planes[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / G;
    const int line = (blockIdx.x * kWarps + warp) * LPW + grp;
    const int w = a.w, h = a.h;

    int dx = 1, dy = 0, x = 0, y = 0, n = 0;
    bool wide = false;
    if (line < total_lines) {
        locate_line(a, line, &dx, &dy, &x, &y);
        const int nx = dx > 0 ? w - x : (dx < 0 ? x + 1 : 0x7FFFFFFF);
        const int ny = dy > 0 ? h - y : (dy < 0 ? y + 1 : 0x7FFFFFFF);
        n = min(nx, ny);
        const uint32_t* f = dy == 0 ? fl.row + y
                                    : (dx == 0 ? fl.col + x : (dx == dy ? fl.diag + (x - y + h - 1) : fl.anti + (x + y)));
        wide = *f != 0u;
    }
    LineCtx lc;
    lc.rec = rec;
    lc.lut = lut;
    lc.gl = lane % G;
    lc.n = n;
    const int nmax = static_cast<int>(__reduce_max_sync(0xFFFFFFFFu, static_cast<unsigned>(n)));
    lc.steps = (nmax + S - 1) / S * S;  // padded: steps past a line's end see empty pixels
    lc.q = y * w + x;
    lc.dp = dy * w + dx;
    lc.dummy = w * h;
    // SN: canonical slot of +-(dx, dy) and the direction's sign (sgm.cpp:72-87)
    const int slot = dy == 0 ? 0 : (dx == 0 ? 1 : (dx == dy ? 2 : 3));
    lc.sign = (dy == 0 || dx == 0) ? dx + dy : dx;
    lc.off_sh = (slot & 1) * 16;
    lc.off_hi = (slot >> 1) != 0;
    lc.planes = s_planes;
    lc.rs = EMB == 0 ? 1 : (EMB == 1 ? 3 : 2);
    lc.x0 = x;
    lc.y0 = y;
    lc.dx = dx;
    lc.dy = dy;

    uint32_t* sA = smem + 256 + (warp * LPW + grp) * stride + kSent;
    uint32_t* sB = sA + PASS + 2 * kSent;
    if (lc.gl < kSent) {
        sA[-kSent + lc.gl] = kSentinel;
        sB[-kSent + lc.gl] = kSentinel;
    }
    if (__any_sync(0xFFFFFFFFu, wide)) {
        uint32_t* bufA = sA;
        uint32_t* bufB = sB;
        if (wide) {
            const size_t gs = static_cast<size_t>(a.pmax) + 2 * kSent;
            bufA = a.scratch + static_cast<size_t>(line) * 2 * gs + kSent;
            bufB = bufA + gs;
            if (lc.gl < kSent) {
                bufA[-kSent + lc.gl] = kSentinel;
                bufB[-kSent + lc.gl] = kSentinel;
            }
        }
        __syncwarp();
        line_steps<SN, G, K, S, GAP, false, 0, AGG16, PG>(a, lc, bufA, bufB);
    } else {
        __syncwarp();
        line_steps<SN, G, K, S, GAP, true, EMB, AGG16, PG>(a, lc, sA, sB);
    }
}

// compute_normal_offsets (sgm.cpp:252-299) on the upscaled prior maps.
constexpr int kOffsetSmemPlanes = 4096;

__global__ void normal_offsets_kernel(OffsetArgs a) {
    using namespace dev;
    // the plane stack in shared memory (binary searches on every pixel's chain)
    extern __shared__ double s_stack[];
    if (a.nplanes <= kOffsetSmemPlanes) {
        for (int i = threadIdx.y * blockDim.x + threadIdx.x; i < a.nplanes; i += blockDim.x * blockDim.y)
            s_stack[i] = a.planes[i];
        a.planes = s_stack;
        __syncthreads();
    }
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
        // the rays of (x, y) and of its 4 canonical predecessors share five
        // coordinate divisions (unproject, geometry.hpp:28-30)
        const D3 r00 = unproject_px(a.intr, x, y), r10 = unproject_px(a.intr, x - 1, y - 1),
                 r01 = unproject_px(a.intr, x, y + 1);
        const double ux0 = r00.x, ux1 = r10.x, uy0 = r00.y, uym = r10.y, uyp = r01.y;
        const D3 ray{ux0, uy0, 1.0};
        const double denom0 = dot3(pn, ray);
        if (!(fabs(denom0) < 1e-12 || div(-1.0, denom0) <= 0.0)) {
            const double delta_anchor = mul(double(depth), -denom0);
            const int i0 = dev::nearest_index(a.planes, a.nplanes, delta_anchor);
            const D3 anchor = scale3(div(-a.planes[i0], denom0), ray);
            const int cd[4][2] = {{1, 0}, {0, 1}, {1, 1}, {1, -1}};
            for (int c = 0; c < 4; ++c) {
                const D3 ray_q{cd[c][0] ? ux1 : ux0, cd[c][1] == 0 ? uy0 : (cd[c][1] > 0 ? uym : uyp), 1.0};
                const double denom_t = dot3(n, ray_q);
                if (fabs(denom_t) < 1e-12)
                    continue;
                const double t = div(dot3(n, anchor), denom_t);
                if (t <= 0.0)
                    continue;
                const double delta_q = -dot3(pn, scale3(t, ray_q));
                if (delta_q <= 0.0)
                    continue;
                double df = sub(fractional_index_from(a.planes, a.nplanes, delta_q, i0), double(i0));
                df = df < -32000.0 ? -32000.0 : (32000.0 < df ? 32000.0 : df);
                o[c] = static_cast<short>(lround(df));
            }
        }
    }
    reinterpret_cast<short4*>(a.out)[p] = out;
}

}  // namespace

// Dynamic shared-memory attributes are set to each kernel's LARGEST possible
// size, a constant: contexts on other host threads launch the same kernels
// with other sizes, and a per-launch setting could shrink the limit between
// another thread's set and launch.
constexpr int kSgmSmemMax = 200 * 1024;  // sgm_kernel: kWarps x 2 x pmax words, pmax <= sgm_smem_pmax_limit()

template <int VARIANT>
void launch_sgm(const SgmArgs& a, int total, int blocks, size_t smem, bool fast32, cudaStream_t s) {
    if (fast32) {
        FMVS_CUDA_CHECK(cudaFuncSetAttribute(sgm_kernel<VARIANT, int>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kSgmSmemMax));
        sgm_kernel<VARIANT, int><<<blocks, kWarps * 32, smem, s>>>(a, total);
    } else {
        FMVS_CUDA_CHECK(cudaFuncSetAttribute(sgm_kernel<VARIANT, long long>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kSgmSmemMax));
        sgm_kernel<VARIANT, long long><<<blocks, kWarps * 32, smem, s>>>(a, total);
    }
}

template <int VARIANT, typename V, int G, int K>
void launch_lanes(const SgmArgs& a, int total, cudaStream_t s) {
    constexpr int LPW = 32 / G;
    const int caps = a.group_caps;
    // line stride = 2 * caps padded so stride % 32 == G % 32: the LPW lines of
    // a warp start in distinct banks
    int stride = 2 * (caps + 2 * kSent);
    stride += ((G % 32) - stride % 32 + 32) % 32;
    const int blocks = (total + kWarps * LPW - 1) / (kWarps * LPW);
    const size_t smem = static_cast<size_t>(kWarps) * LPW * stride * sizeof(uint32_t);
    // largest: group_caps <= 1024 with one line per warp (dense coarsest
    // levels), 32 otherwise (refined levels, stage API)
    constexpr int kCapsMax = G == 32 ? 1024 : 32;
    if (caps > kCapsMax)
        throw Error(FMVS_ERR_CONFIG, "sgm: path buffer capacity exceeds the kernel's shared memory");
    const int smem_max = kWarps * LPW * (2 * (kCapsMax + 2 * kSent) + 32) * static_cast<int>(sizeof(uint32_t));
    FMVS_CUDA_CHECK(cudaFuncSetAttribute(sgm_lanes_kernel<VARIANT, V, G, K>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    sgm_lanes_kernel<VARIANT, V, G, K><<<blocks, kWarps * 32, smem, s>>>(a, total, caps, stride);
}

template <int VARIANT, typename V>
void launch_group_g(const SgmArgs& a, int total, cudaStream_t s) {
    const int g = a.group, k = a.kper;
    if (g == 4 && (k == 4 || k == 3))  // K = 3 is a line-kernel blocking
        launch_lanes<VARIANT, V, 4, 4>(a, total, s);
    else if (g == 8 && k == 2)
        launch_lanes<VARIANT, V, 8, 2>(a, total, s);
    else if (g == 8 && k == 4)
        launch_lanes<VARIANT, V, 8, 4>(a, total, s);
    else if (g == 32 && k == 1)
        launch_lanes<VARIANT, V, 32, 1>(a, total, s);
    else if (g == 32 && k == 4)
        launch_lanes<VARIANT, V, 32, 4>(a, total, s);
    else if (g == 32 && k == 8)
        launch_lanes<VARIANT, V, 32, 8>(a, total, s);
    else
        throw Error(FMVS_ERR_CONFIG, "sgm: unsupported lane blocking");
}

template <bool SN, bool PG, int G, int K, int S, int GAP>
void launch_line_sg(const SgmArgs& a, int total, cudaStream_t s) {
    constexpr int LPW = 32 / G;
    // a line is narrow when every pixel fits one pass (its shared buffers
    // hold G*K slots); wider lines run from their global scratch
    const int caps = G * K;
    int stride = 2 * (caps + 2 * kSent);
    stride += ((G % 32) - stride % 32 + 32) % 32;
    const int blocks = (total + kWarps * LPW - 1) / (kWarps * LPW);
    const size_t smem = (256 + static_cast<size_t>(kWarps) * LPW * stride + 1) * sizeof(uint32_t) +
                        (PG ? static_cast<size_t>(a.nplanes) * sizeof(double) : 0);
    auto* rec = reinterpret_cast<uint4*>(a.line_scratch);
    const LineFlags fl = line_flags(a.line_scratch + kRecWords * (static_cast<size_t>(a.w) * a.h + 1), a.w, a.h);
    FMVS_CUDA_CHECK(cudaMemsetAsync(fl.row, 0, line_flag_words(a.w, a.h) * sizeof(uint32_t), s));
    const int npx = a.w * a.h + 1;
    // embedded costs (G = 4, K <= 4; FMVS_SGM_EMB=0 keeps them in the volume)
    static const bool emb_on = [] {
        const char* e = std::getenv("FMVS_SGM_EMB");
        return !(e && e[0] == '0');
    }();
    // 10-bit packing when every cost of the volume is < 1024 (the host's
    // bound, SgmArgs::cost_max) and a lane holds <= 3 hypotheses
    constexpr int kEmb = (G == 4 && K <= 4) ? ((K <= 3) ? 2 : 1) : 0;
    const int emb = !emb_on ? 0 : (kEmb == 2 && !(a.cost_max >= 0 && a.cost_max < 1024) ? 1 : kEmb);
    sgm_prep_kernel<<<(npx + 255) / 256, 256, 0, s>>>(a, rec, fl, caps, emb);
    // the attribute is set to this instantiation's largest possible size (a
    // constant: contexts on other host threads launch the same kernel)
    const int smem_max = static_cast<int>((256 + static_cast<size_t>(kWarps) * LPW * stride + 1) *
                                              sizeof(uint32_t) +
                                          (PG ? static_cast<size_t>(kRecPlanes) * sizeof(double) : 0));
    auto go = [&](auto kernel) {
        FMVS_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
        kernel<<<blocks, kWarps * 32, smem, s>>>(a, rec, fl, total, stride);
    };
    constexpr int kEmb1 = kEmb ? 1 : 0;
    if (emb == 2 && a.agg16)
        go(sgm_line_kernel<SN, G, K, S, GAP, kEmb, true, PG>);
    else if (emb == 2)
        go(sgm_line_kernel<SN, G, K, S, GAP, kEmb, false, PG>);
    else if (emb == 1 && a.agg16)
        go(sgm_line_kernel<SN, G, K, S, GAP, kEmb1, true, PG>);
    else if (emb == 1)
        go(sgm_line_kernel<SN, G, K, S, GAP, kEmb1, false, PG>);
    else if (a.agg16)
        go(sgm_line_kernel<SN, G, K, S, GAP, 0, true, PG>);
    else
        go(sgm_line_kernel<SN, G, K, S, GAP, 0, false, PG>);
}

// Pipeline depth S (pixels whose records are in registers; measured 6 / 8 /
// 10 / 12 at C2 L0: 8 best) and GAP (steps between a pixel's record and its
// cost loads when the costs are not embedded).
template <bool SN, bool PG, int G, int K>
void launch_line(const SgmArgs& a, int total, cudaStream_t s) {
    if constexpr (K >= 8)
        launch_line_sg<SN, PG, G, K, 4, 1>(a, total, s);
    else
        launch_line_sg<SN, PG, G, K, 8, 3>(a, total, s);
}

template <bool SN, bool PG>
bool launch_line_gk(const SgmArgs& a, int total, cudaStream_t s) {
    if (a.group == 4 && a.kper == 4)
        launch_line<SN, PG, 4, 4>(a, total, s);
    else if (a.group == 4 && a.kper == 3)
        launch_line<SN, PG, 4, 3>(a, total, s);
    else if (a.group == 32 && a.kper == 4)
        launch_line<SN, PG, 32, 4>(a, total, s);
    else if (a.group == 32 && a.kper == 8)
        launch_line<SN, PG, 32, 8>(a, total, s);
    else
        return false;
    return true;
}

size_t sgm_line_scratch_words(int w, int h) {
    return static_cast<size_t>(kRecWords) * (static_cast<size_t>(w) * h + 1) + line_flag_words(w, h);
}

bool sgm_fast32(const SgmArgs& a) {
    return a.phi1 >= 0 && a.phi2_max >= 0 && a.phi1 < (1ll << 28) && a.phi2_max < (1ll << 28);
}

bool sgm_line_applicable(const SgmArgs& a) {
    // line kernel: any variant, int32, unit directions, 32-bit entry indices
    static const bool line_on = [] {
        const char* e = std::getenv("FMVS_SGM_LINE");
        return !(e && e[0] == '0');
    }();
    bool unit = true;
    for (int d = 0; d < a.ndirs; ++d)
        unit = unit && std::abs(a.dirs[d][0]) <= 1 && std::abs(a.dirs[d][1]) <= 1 &&
               (a.dirs[d][0] != 0 || a.dirs[d][1] != 0);
    const bool gk = (a.group == 4 && (a.kper == 3 || a.kper == 4)) ||
                    (a.group == 32 && (a.kper == 4 || a.kper == 8));
    return line_on && a.line_scratch && a.scratch && sgm_fast32(a) && unit && gk && a.nplanes <= kRecPlanes &&
           a.entries_bound + 1024 < (1ull << 32);
}

bool sgm_agg16_ok(const SgmArgs& a, long long cost_max) {
    // every path value lies in [0, cost + phi2_max] (its best candidate is at
    // most prev_min + phi2), so the aggregate of `ndirs` paths stays below
    // ndirs * (cost_max + phi2_max): two aggregates per 32-bit word never carry
    return sgm_line_applicable(a) && cost_max >= 0 &&
           static_cast<long long>(a.ndirs) * (cost_max + a.phi2_max) < 65536;
}

void sgm(const SgmArgs& a, cudaStream_t s) {
    const int total = sgm_lines(a.w, a.h, a.dirs, a.ndirs);
    if (total == 0)
        return;
    // int32 recurrence is exact when every intermediate stays below 2^31:
    // path values <= 65535 + phi2_max, candidates <= value + max(phi1, phi2).
    const bool fast32 = sgm_fast32(a);
    static_assert(kAggSlack >= 32 * 8, "inactive lanes of a pass add 0 up to G*K - 1 entries past a pixel");
    if (sgm_line_applicable(a)) {
        if (a.variant == FMVS_SGM_PATH_GRADIENT)
            launch_line_gk<false, true>(a, total, s);
        else if (a.offsets)
            launch_line_gk<true, false>(a, total, s);
        else
            launch_line_gk<false, false>(a, total, s);
        FMVS_CUDA_CHECK(cudaGetLastError());
        return;
    }
    if (a.agg16)
        throw Error(FMVS_ERR_CONFIG, "sgm: packed u16 aggregate needs the line kernel");
    if (a.group > 0) {
        // lane-blocked kernel; scratch (global overflow buffers) is mandatory here
        if (a.variant == FMVS_SGM_PATH_GRADIENT) {
            if (fast32)
                launch_group_g<FMVS_SGM_PATH_GRADIENT, int>(a, total, s);
            else
                launch_group_g<FMVS_SGM_PATH_GRADIENT, long long>(a, total, s);
        } else if (a.variant == FMVS_SGM_SURFACE_NORMAL) {
            if (fast32)
                launch_group_g<FMVS_SGM_SURFACE_NORMAL, int>(a, total, s);
            else
                launch_group_g<FMVS_SGM_SURFACE_NORMAL, long long>(a, total, s);
        } else {
            if (fast32)
                launch_group_g<FMVS_SGM_PLANE, int>(a, total, s);
            else
                launch_group_g<FMVS_SGM_PLANE, long long>(a, total, s);
        }
        FMVS_CUDA_CHECK(cudaGetLastError());
        return;
    }
    const int blocks = (total + kWarps - 1) / kWarps;
    const size_t smem = a.scratch ? 0 : static_cast<size_t>(kWarps) * 2 * a.pmax * sizeof(uint32_t);
    switch (a.variant) {
        case FMVS_SGM_SURFACE_NORMAL:
            launch_sgm<FMVS_SGM_SURFACE_NORMAL>(a, total, blocks, smem, fast32, s);
            break;
        case FMVS_SGM_PATH_GRADIENT:
            launch_sgm<FMVS_SGM_PATH_GRADIENT>(a, total, blocks, smem, fast32, s);
            break;
        default:
            launch_sgm<FMVS_SGM_PLANE>(a, total, blocks, smem, fast32, s);
            break;
    }
    FMVS_CUDA_CHECK(cudaGetLastError());
}

int sgm_total_lines(int w, int h, int ndirs) {
    return ndirs == 8 ? 2 * h + 2 * w + 4 * (w + h - 1) : 2 * h + 2 * w;
}

int sgm_lines(int w, int h, const int (*dirs)[2], int ndirs) {
    int total = 0;
    for (int d = 0; d < ndirs; ++d)
        total += lines_of_dir(w, h, dirs[d][0], dirs[d][1]);
    return total;
}

// Largest per-warp path buffer that keeps kWarps warps in shared memory.
int sgm_smem_pmax_limit() { return (200 * 1024) / (kWarps * 2 * 4); }

void normal_offsets(const OffsetArgs& a, cudaStream_t s) {
    const dim3 block(32, 8);
    const dim3 grid((a.w + 31) / 32, (a.h + 7) / 8);
    const size_t smem = a.nplanes <= kOffsetSmemPlanes ? sizeof(double) * a.nplanes : 0;
    // <= 32 KB: within the default dynamic shared-memory limit (no attribute
    // call -- concurrent host threads would race on a per-launch setting)
    normal_offsets_kernel<<<grid, block, smem, s>>>(a);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

}  // namespace k
}  // namespace fmvs
