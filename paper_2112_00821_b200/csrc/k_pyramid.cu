// K1: image pyramid (blur_and_halve, pipeline.cpp:79-89 over gaussian_blur,
// pipeline.cpp:32-75) and the quad-packed sampling images for the sweep.
//
// blur_and_halve only keeps the blurred image at even (2x, 2y), so each
// output pixel evaluates the three horizontal passes it needs (rows 2y-1..2y+1,
// column 2x, each stored as float like the reference's tmp raster) and the
// vertical pass, all in the reference's FP64 accumulation order
// (acc = 0; acc += k[i] * v for i = -1..1), then lround -> clamp -> u8.
// HBM-bound: 4 B read (L1/L2 reuse) + 1 B written per output pixel.
#include "host.hpp"
#include "kernels.hpp"

namespace fmvs {
namespace k {

namespace {

__device__ __forceinline__ int reflect(int i, int n) {  // pipeline.cpp:44-54
    if (n == 1)
        return 0;
    while (i < 0 || i >= n) {
        if (i < 0)
            i = -i;
        if (i >= n)
            i = 2 * (n - 1) - i;
    }
    return i;
}

__global__ void blur_halve_kernel(const uint8_t* __restrict__ in, int win, int hin,
                                  uint8_t* __restrict__ out, int wout, int hout, double k0,
                                  double k1, double k2) {
    using namespace dev;
    const double c_k3[3] = {k0, k1, k2};
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= wout || y >= hout)
        return;
    const int X = 2 * x, Y = 2 * y;
    const int xm = reflect(X - 1, win), xp = reflect(X + 1, win);
    float tmp[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const int yy = reflect(Y + j - 1, hin);
        const uint8_t* row = in + static_cast<size_t>(yy) * win;
        double acc = 0.0;
        acc = add(acc, mul(c_k3[0], double(__ldg(row + xm))));
        acc = add(acc, mul(c_k3[1], double(__ldg(row + X))));
        acc = add(acc, mul(c_k3[2], double(__ldg(row + xp))));
        tmp[j] = __double2float_rn(acc);
    }
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j)
        acc = add(acc, mul(c_k3[j], double(tmp[j])));
    const float blurred = __double2float_rn(acc);
    long v = lroundf(blurred);
    v = v < 0 ? 0 : (v > 255 ? 255 : v);
    out[static_cast<size_t>(y) * wout + x] = static_cast<uint8_t>(v);
}

__global__ void pack_quads_kernel(const uint8_t* __restrict__ img, int w, int h,
                                  uint32_t* __restrict__ quad) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    const int x1 = min(x + 1, w - 1), y1 = min(y + 1, h - 1);
    const uint8_t* r0 = img + static_cast<size_t>(y) * w;
    const uint8_t* r1 = img + static_cast<size_t>(y1) * w;
    quad[static_cast<size_t>(y) * w + x] = uint32_t(__ldg(r0 + x)) | (uint32_t(__ldg(r0 + x1)) << 8) |
                                           (uint32_t(__ldg(r1 + x)) << 16) |
                                           (uint32_t(__ldg(r1 + x1)) << 24);
}

// Batched forms: blockIdx.z selects the image (one launch for all views of a
// pyramid level / all quad images of a bundle instead of one per image).
__global__ void blur_halve_batch_kernel(ImgBatch b, double k0, double k1, double k2) {
    const ImgJob& j = b.job[blockIdx.z];
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= j.wout || y >= j.hout)
        return;
    using namespace dev;
    const double c_k3[3] = {k0, k1, k2};
    const int X = 2 * x, Y = 2 * y;
    const int xm = reflect(X - 1, j.win), xp = reflect(X + 1, j.win);
    float tmp[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const int yy = reflect(Y + r - 1, j.hin);
        const uint8_t* row = j.in + static_cast<size_t>(yy) * j.win;
        double acc = 0.0;
        acc = add(acc, mul(c_k3[0], double(__ldg(row + xm))));
        acc = add(acc, mul(c_k3[1], double(__ldg(row + X))));
        acc = add(acc, mul(c_k3[2], double(__ldg(row + xp))));
        tmp[r] = __double2float_rn(acc);
    }
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < 3; ++r)
        acc = add(acc, mul(c_k3[r], double(tmp[r])));
    long v = lroundf(__double2float_rn(acc));
    v = v < 0 ? 0 : (v > 255 ? 255 : v);
    j.out[static_cast<size_t>(y) * j.wout + x] = static_cast<uint8_t>(v);
}

// Four quads per thread from two aligned 32-bit row loads (+ the byte right
// of them) and byte permutes, written as one 16-byte store; images whose
// rows or buffers are not 4 / 16-byte aligned take the per-pixel path.
__global__ void pack_quads_batch_kernel(ImgBatch b) {
    const ImgJob& j = b.job[blockIdx.z];
    const int w = j.win, h = j.hin;
    const bool vec = (w & 3) == 0 && (reinterpret_cast<uintptr_t>(j.in) & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(j.quad) & 15) == 0;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (vec) {
        const int x0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
        if (x0 >= w || y >= h)
            return;
        const int y1 = min(y + 1, h - 1);
        const uint8_t* r0 = j.in + static_cast<size_t>(y) * w;
        const uint8_t* r1 = j.in + static_cast<size_t>(y1) * w;
        const uint32_t a = __ldg(reinterpret_cast<const uint32_t*>(r0 + x0));
        const uint32_t c = __ldg(reinterpret_cast<const uint32_t*>(r1 + x0));
        const int xr = min(x0 + 4, w - 1);  // x1 of the group's last pixel (edge clamp)
        const uint32_t a4 = __ldg(r0 + xr), c4 = __ldg(r1 + xr);
        uint32_t q[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t top = __byte_perm(a, a4, static_cast<uint32_t>(k | ((k + 1) << 4)));
            const uint32_t bot = __byte_perm(c, c4, static_cast<uint32_t>(k | ((k + 1) << 4)));
            q[k] = __byte_perm(top, bot, 0x5410);
        }
        *reinterpret_cast<uint4*>(j.quad + static_cast<size_t>(y) * w + x0) = make_uint4(q[0], q[1], q[2], q[3]);
        return;
    }
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= j.win || y >= j.hin)
        return;
    const int x1 = min(x + 1, w - 1), y1 = min(y + 1, h - 1);
    const uint8_t* r0 = j.in + static_cast<size_t>(y) * w;
    const uint8_t* r1 = j.in + static_cast<size_t>(y1) * w;
    j.quad[static_cast<size_t>(y) * w + x] = uint32_t(__ldg(r0 + x)) | (uint32_t(__ldg(r0 + x1)) << 8) |
                                             (uint32_t(__ldg(r1 + x)) << 16) |
                                             (uint32_t(__ldg(r1 + x1)) << 24);
}

}  // namespace

void blur_halve_batch(const ImgBatch& b, int n, const double k3[3], cudaStream_t s) {
    int mw = 1, mh = 1;
    for (int i = 0; i < n; ++i) {
        mw = max(mw, b.job[i].wout);
        mh = max(mh, b.job[i].hout);
    }
    blur_halve_batch_kernel<<<dim3((mw + 31) / 32, (mh + 7) / 8, n), dim3(32, 8), 0, s>>>(b, k3[0], k3[1], k3[2]);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void pack_quads_batch(const ImgBatch& b, int n, cudaStream_t s) {
    int mw = 1, mh = 1;
    for (int i = 0; i < n; ++i) {
        const ImgJob& j = b.job[i];
        const bool vec = (j.win & 3) == 0 && (reinterpret_cast<uintptr_t>(j.in) & 3) == 0 &&
                         (reinterpret_cast<uintptr_t>(j.quad) & 15) == 0;
        mw = max(mw, vec ? j.win / 4 : j.win);  // threads along x (4 pixels each when vec)
        mh = max(mh, j.hin);
    }
    pack_quads_batch_kernel<<<dim3((mw + 31) / 32, (mh + 7) / 8, n), dim3(32, 8), 0, s>>>(b);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void blur_halve(const uint8_t* in, int win, int hin, uint8_t* out, int wout, int hout,
                const double k3[3], cudaStream_t s) {
    const dim3 block(32, 8);
    const dim3 grid((wout + 31) / 32, (hout + 7) / 8);
    blur_halve_kernel<<<grid, block, 0, s>>>(in, win, hin, out, wout, hout, k3[0], k3[1], k3[2]);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void pack_quads(const uint8_t* img, int w, int h, uint32_t* quad, cudaStream_t s) {
    const dim3 block(32, 8);
    const dim3 grid((w + 31) / 32, (h + 7) / 8);
    pack_quads_kernel<<<grid, block, 0, s>>>(img, w, h, quad);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

}  // namespace k
}  // namespace fmvs
