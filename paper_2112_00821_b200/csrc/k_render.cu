// Synthetic input generator on the device: render_scene (render.cpp:52-141)
// for any set of textured planes with extents, checkerboard or fractal
// value-noise texture (render.cpp:12-50). Used by bench.py to produce the
// BASELINE configs' bundles at full resolution without a CPU bottleneck;
// parity with the reference renderer: tests/test_fullsize_gpu.py
// (test_render_fullsize) and tests/test_parity_gpu.py (test_render_*).
#include "host.hpp"
#include "kernels.hpp"

namespace fmvs {
namespace k {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

__device__ __forceinline__ double lattice(int64_t ix, int64_t iy, uint64_t seed) {
    const uint64_t hsh = splitmix64(static_cast<uint64_t>(ix) * 0x8da6b343ULL ^
                                    static_cast<uint64_t>(iy) * 0xd8163841ULL ^ seed);
    return dev::mul(double(hsh >> 11), 0x1.0p-53);
}

__device__ double octave(double u, double v, uint64_t seed) {
    using namespace dev;
    const double fu = floor(u), fv = floor(v);
    const int64_t iu = static_cast<int64_t>(fu), iv = static_cast<int64_t>(fv);
    double au = sub(u, fu), av = sub(v, fv);
    au = mul(mul(au, au), sub(3.0, mul(2.0, au)));
    av = mul(mul(av, av), sub(3.0, mul(2.0, av)));
    const double v00 = lattice(iu, iv, seed), v10 = lattice(iu + 1, iv, seed);
    const double v01 = lattice(iu, iv + 1, seed), v11 = lattice(iu + 1, iv + 1, seed);
    const double omu = sub(1.0, au);
    return add(mul(sub(1.0, av), add(mul(omu, v00), mul(au, v10))),
               mul(av, add(mul(omu, v01), mul(au, v11))));
}

__device__ double value_noise(double u, double v, uint64_t seed) {
    using namespace dev;
    double sum = 0.0, amp = 1.0, total = 0.0, freq = 1.0;
    for (int o = 0; o < 3; ++o) {
        sum = add(sum, mul(amp, octave(mul(u, freq), mul(v, freq), seed + o)));
        total = add(total, amp);
        amp = mul(amp, 0.5);
        freq = mul(freq, 2.0);
    }
    return div(sum, total);
}

__global__ void render_kernel(RenderArgs a) {
    using namespace dev;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= a.w || y >= a.h)
        return;
    const size_t p = static_cast<size_t>(y) * a.w + x;
    const D3 ray = unproject(a.intr, double(x), double(y));
    // dir = R^T * ray
    const D3 dir{add(add(mul(a.rot[0], ray.x), mul(a.rot[3], ray.y)), mul(a.rot[6], ray.z)),
                 add(add(mul(a.rot[1], ray.x), mul(a.rot[4], ray.y)), mul(a.rot[7], ray.z)),
                 add(add(mul(a.rot[2], ray.x), mul(a.rot[5], ray.y)), mul(a.rot[8], ray.z))};
    const D3 c{a.center[0], a.center[1], a.center[2]};
    // nearest plane hit inside its extents (render.cpp:85-110)
    double best_t = __longlong_as_double(0x7FF0000000000000LL);  // +inf
    int best = -1;
    double best_u = 0.0, best_v = 0.0;
    for (int pi = 0; pi < a.nplanes; ++pi) {
        const RenderPlane& f = a.planes[pi];
        const D3 n{f.n[0], f.n[1], f.n[2]};
        const double denom = dot3(n, dir);
        if (fabs(denom) < 1e-12)
            continue;
        const double t = div(dot3(n, sub3(D3{f.pt[0], f.pt[1], f.pt[2]}, c)), denom);
        if (t <= 0.0 || t >= best_t)
            continue;
        const D3 hit = add3(c, scale3(t, dir));
        const D3 rel = sub3(hit, D3{f.pt[0], f.pt[1], f.pt[2]});
        const double pu = dot3(rel, D3{f.u[0], f.u[1], f.u[2]});
        const double pv = dot3(rel, D3{f.v[0], f.v[1], f.v[2]});
        if (fabs(pu) > f.ext_u || fabs(pv) > f.ext_v)
            continue;
        best_t = t;
        best = pi;
        best_u = pu;
        best_v = pv;
    }
    uint8_t pix = 0;
    float gd = 0.0f;
    float3 gn = make_float3(0.0f, 0.0f, 0.0f);
    if (best >= 0) {
        const double tu = div(best_u, a.texture_scale), tv = div(best_v, a.texture_scale);
        double val;
        if (a.texture == FMVS_TEXTURE_CHECKERBOARD) {  // render.cpp:118-121
            const long long parity = static_cast<long long>(floor(tu)) + static_cast<long long>(floor(tv));
            val = (parity & 1) ? 224.0 / 255.0 : 32.0 / 255.0;
        } else {
            val = value_noise(tu, tv, a.seed + 7919ull * static_cast<uint64_t>(best));
        }
        pix = static_cast<uint8_t>(lround(mul(255.0, val)));
        gd = __double2float_rn(best_t);
        // n_cam = R * n, camera-facing
        const RenderPlane& f = a.planes[best];
        const D3 n{f.n[0], f.n[1], f.n[2]};
        D3 nc{add(add(mul(a.rot[0], n.x), mul(a.rot[1], n.y)), mul(a.rot[2], n.z)),
              add(add(mul(a.rot[3], n.x), mul(a.rot[4], n.y)), mul(a.rot[5], n.z)),
              add(add(mul(a.rot[6], n.x), mul(a.rot[7], n.y)), mul(a.rot[8], n.z))};
        if (nc.z > 0.0)
            nc = {-nc.x, -nc.y, -nc.z};
        gn = make_float3(__double2float_rn(nc.x), __double2float_rn(nc.y), __double2float_rn(nc.z));
    }
    a.image[p] = pix;
    if (a.gt_depth)
        a.gt_depth[p] = gd;
    if (a.gt_normals) {
        a.gt_normals[3 * p] = gn.x;
        a.gt_normals[3 * p + 1] = gn.y;
        a.gt_normals[3 * p + 2] = gn.z;
    }
}

}  // namespace

void render_view(const RenderArgs& a, cudaStream_t s) {
    render_kernel<<<dim3((a.w + 31) / 32, (a.h + 7) / 8), dim3(32, 8), 0, s>>>(a);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

}  // namespace k
}  // namespace fmvs
