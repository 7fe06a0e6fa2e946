// Output stage of the CLI: the 8-bit visualisations of
// colorize.cpp (viridis depth :32-43, (n+1)/2 normals :45-57, gray
// confidence :59-70), one thread per pixel, in the reference's mixed
// float/double expression order so the bytes are identical. HBM-bound:
// 4-12 B in, 3 B out per pixel.
#include "host.hpp"
#include "kernels.hpp"

namespace fmvs {
namespace k {

namespace {

__constant__ double c_viridis[9][3] = {  // colorize.cpp:11-16
    {0.267004, 0.004874, 0.329415}, {0.282623, 0.140926, 0.457517},
    {0.253935, 0.265254, 0.529983}, {0.206756, 0.371758, 0.553117},
    {0.163625, 0.471133, 0.558148}, {0.127568, 0.566949, 0.550556},
    {0.134692, 0.658636, 0.517649}, {0.477504, 0.821444, 0.318195},
    {0.993248, 0.906157, 0.143936}};

__device__ __forceinline__ uint8_t lround_u8(double v) { return static_cast<uint8_t>(lround(v)); }

__global__ void colorize_depth_kernel(const float* __restrict__ d, int n, double lo, double span,
                                      uint8_t* __restrict__ rgb) {
    using namespace dev;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n)
        return;
    uint8_t c3[3] = {0, 0, 0};
    const float v = d[p];
    if (depth_ok(v)) {
        double t = div(sub(double(v), lo), span);  // (d - lo) / span (:39-40)
        t = t < 0.0 ? 0.0 : (1.0 < t ? 1.0 : t);   // viridis (:18-28)
        const double pos = mul(t, 8.0);
        const int i = min(static_cast<int>(pos), 7);
        const double a = sub(pos, double(i));
        for (int c = 0; c < 3; ++c)
            c3[c] = lround_u8(mul(255.0, add(mul(sub(1.0, a), c_viridis[i][c]), mul(a, c_viridis[i + 1][c]))));
    }
    rgb[3 * p] = c3[0];
    rgb[3 * p + 1] = c3[1];
    rgb[3 * p + 2] = c3[2];
}

__global__ void colorize_normals_kernel(const float* __restrict__ nrm, int n, uint8_t* __restrict__ rgb) {
    using namespace dev;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n)
        return;
    const float x = nrm[3 * p], y = nrm[3 * p + 1], z = nrm[3 * p + 2];
    uint8_t c3[3] = {0, 0, 0};
    if (normal_ok(x, y, z)) {
        const float v[3] = {x, y, z};
        for (int c = 0; c < 3; ++c) {
            float f = __fdiv_rn(__fadd_rn(v[c], 1.0f), 2.0f);  // (n[c] + 1.0f) / 2.0f (:53-54)
            f = f < 0.0f ? 0.0f : (1.0f < f ? 1.0f : f);
            c3[c] = lround_u8(mul(255.0, double(f)));
        }
    }
    rgb[3 * p] = c3[0];
    rgb[3 * p + 1] = c3[1];
    rgb[3 * p + 2] = c3[2];
}

__global__ void colorize_conf_kernel(const float* __restrict__ cf, int n, uint8_t* __restrict__ rgb) {
    using namespace dev;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n)
        return;
    const float c = cf[p];
    uint8_t v = 0;
    if (c > 0.0f) {  // :64-67
        const float cc = c < 0.0f ? 0.0f : (1.0f < c ? 1.0f : c);
        v = lround_u8(mul(255.0, double(cc)));
    }
    rgb[3 * p] = v;
    rgb[3 * p + 1] = v;
    rgb[3 * p + 2] = v;
}

}  // namespace

void colorize(int kind, const float* in, int n, double lo, double hi, uint8_t* rgb, cudaStream_t s) {
    if (n <= 0)
        return;
    const int b = 256, g = (n + b - 1) / b;
    if (kind == 0)
        colorize_depth_kernel<<<g, b, 0, s>>>(in, n, lo, hi > lo ? hi - lo : 1.0, rgb);
    else if (kind == 1)
        colorize_normals_kernel<<<g, b, 0, s>>>(in, n, rgb);
    else
        colorize_conf_kernel<<<g, b, 0, s>>>(in, n, rgb);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

}  // namespace k
}  // namespace fmvs
