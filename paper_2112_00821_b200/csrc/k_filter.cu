// Post-filters of the per-frame maps: the DoG texture
// mask (dog_mask, postfilter.cpp:67-79 with remove_speckles :14-51 and
// dilate_3x3 :53-63 over gaussian_blur, pipeline.cpp:32-75), apply_mask
// (:81-93) and the multi-view geometric consistency mask
// (geometric_consistency_mask, :95-160).
//
// * Blur: separable, reflected borders, FP64 accumulation in the reference's
//   tap order, the horizontal pass stored as float (pipeline.cpp:58-75).
// * Speckle removal: 8-connected components by a global union-find (labels
//   only decrease through atomicMin, so every component converges to its
//   minimum pixel index), path compression, size counting with integer
//   atomics, then flipping components smaller than the threshold. The
//   component partition is unique, so the mask is bit-identical to the
//   reference's sequential flood fill.
// * Geometric consistency: thread per reference pixel, the reference's FP64
//   expression order (shim order, IEEE intrinsics, no FMA).
// All kernels are HBM/L2-bound per-pixel passes (a few bytes per pixel).
#include "host.hpp"
#include "kernels.hpp"

namespace fmvs {
namespace k {

namespace {

__device__ __forceinline__ int reflect_i(int i, int n) {  // pipeline.cpp:44-54
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

dim3 grid2(int w, int h) { return dim3((w + 31) / 32, (h + 7) / 8); }

__global__ void blur_rows_kernel(const uint8_t* __restrict__ img, int w, int h, BlurKernel k,
                                 float* __restrict__ tmp) {
    using namespace dev;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    const uint8_t* row = img + static_cast<size_t>(y) * w;
    double acc = 0.0;
    for (int i = -k.radius; i <= k.radius; ++i)
        acc = add(acc, mul(k.w[i + k.radius], double(__ldg(row + reflect_i(x + i, w)))));
    tmp[static_cast<size_t>(y) * w + x] = __double2float_rn(acc);
}

// vertical pass fused with the DoG activation threshold (postfilter.cpp:70-74)
__global__ void blur_cols_dog_kernel(const float* __restrict__ tmp, const uint8_t* __restrict__ img,
                                     int w, int h, BlurKernel k, uint8_t* __restrict__ mask) {
    using namespace dev;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    double acc = 0.0;
    for (int i = -k.radius; i <= k.radius; ++i)
        acc = add(acc, mul(k.w[i + k.radius],
                           double(__ldg(tmp + static_cast<size_t>(reflect_i(y + i, h)) * w + x))));
    const float smooth = __double2float_rn(acc);
    const size_t p = static_cast<size_t>(y) * w + x;
    mask[p] = fabsf(__fsub_rn(float(img[p]), smooth)) > 0.5f ? 1 : 0;
}

__global__ void blur_cols_kernel(const float* __restrict__ tmp, int w, int h, BlurKernel k,
                                 float* __restrict__ out) {
    using namespace dev;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    double acc = 0.0;
    for (int i = -k.radius; i <= k.radius; ++i)
        acc = add(acc, mul(k.w[i + k.radius],
                           double(__ldg(tmp + static_cast<size_t>(reflect_i(y + i, h)) * w + x))));
    out[static_cast<size_t>(y) * w + x] = __double2float_rn(acc);
}

// census_transform / census_bits_at (matching.cpp:28-55): neighbour < centre,
// row-major, MSB first, centre skipped, edge-clamped.
__global__ void census_kernel(const uint8_t* __restrict__ img, int w, int h, int ww, int wh,
                              uint64_t* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    const int rx = ww / 2, ry = wh / 2;
    const uint8_t c = img[static_cast<size_t>(y) * w + x];
    uint64_t bits = 0;
    for (int dy = -ry; dy <= ry; ++dy)
        for (int dx = -rx; dx <= rx; ++dx) {
            if (dx == 0 && dy == 0)
                continue;
            const int xx = min(max(x + dx, 0), w - 1), yy = min(max(y + dy, 0), h - 1);
            bits = (bits << 1) | (__ldg(img + static_cast<size_t>(yy) * w + xx) < c ? 1u : 0u);
        }
    out[static_cast<size_t>(y) * w + x] = bits;
}

__device__ __forceinline__ int uf_find(const int* labels, int p) {
    for (;;) {
        const int q = __ldcg(labels + p);
        if (q == p)
            return p;
        p = q;
    }
}

// Union of the trees of a and b: the larger root is hooked under the smaller
// one with atomicMin; a failed hook (the root changed concurrently) retries
// from the value found there.
__device__ void uf_union(int* labels, int a, int b) {
    for (;;) {
        a = uf_find(labels, a);
        b = uf_find(labels, b);
        if (a == b)
            return;
        if (a < b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicMin(labels + a, b);
        if (old == a)
            return;
        a = old;
    }
}

__global__ void ccl_init_kernel(const uint8_t* __restrict__ mask, int w, int h, uint8_t value,
                                int* __restrict__ labels, int* __restrict__ sizes) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    const int p = y * w + x;
    labels[p] = mask[p] == value ? p : -1;
    sizes[p] = 0;
}

__global__ void ccl_merge_kernel(const uint8_t* __restrict__ mask, int w, int h, uint8_t value,
                                 int* labels) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    const int p = y * w + x;
    if (mask[p] != value)
        return;
    // half of the 8-neighbourhood: E, SW, S, SE (the other half is covered
    // by the neighbours' own passes)
    if (x + 1 < w && mask[p + 1] == value)
        uf_union(labels, p, p + 1);
    if (y + 1 < h) {
        if (x > 0 && mask[p + w - 1] == value)
            uf_union(labels, p, p + w - 1);
        if (mask[p + w] == value)
            uf_union(labels, p, p + w);
        if (x + 1 < w && mask[p + w + 1] == value)
            uf_union(labels, p, p + w + 1);
    }
}

__global__ void ccl_count_kernel(int w, int h, int* labels, int* sizes) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    const int p = y * w + x;
    if (labels[p] < 0)
        return;
    const int r = uf_find(labels, p);
    atomicAdd(sizes + r, 1);
}

__global__ void ccl_flip_kernel(uint8_t* mask, int w, int h, uint8_t value, const int* labels,
                                const int* sizes, int min_size) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    const int p = y * w + x;
    if (labels[p] < 0)
        return;
    if (sizes[uf_find(labels, p)] < min_size)
        mask[p] = value ? 0 : 1;
}

__global__ void dilate3_kernel(const uint8_t* __restrict__ in, int w, int h,
                               uint8_t* __restrict__ out) {  // postfilter.cpp:53-63
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    uint8_t v = 0;
    for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
            const int xx = x + dx, yy = y + dy;
            if (xx >= 0 && yy >= 0 && xx < w && yy < h && in[yy * w + xx])
                v = 1;
        }
    out[y * w + x] = v;
}

__global__ void apply_mask_kernel(float* depth, float* normals_xyz, float* conf,
                                  const uint8_t* __restrict__ mask, int n) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n || mask[p])
        return;
    depth[p] = 0.0f;  // postfilter.cpp:88-91
    normals_xyz[3 * p] = 0.0f;
    normals_xyz[3 * p + 1] = 0.0f;
    normals_xyz[3 * p + 2] = 0.0f;
    conf[p] = 0.0f;
}

using dev::D3;

// Pose::to_world: rotation^T * xc + center (geometry.hpp:52-53), each row of
// the product reduced left to right.
__device__ __forceinline__ D3 to_world(const double* R, const double* C, D3 v) {
    using namespace dev;
    return {add(add(add(mul(R[0], v.x), mul(R[3], v.y)), mul(R[6], v.z)), C[0]),
            add(add(add(mul(R[1], v.x), mul(R[4], v.y)), mul(R[7], v.z)), C[1]),
            add(add(add(mul(R[2], v.x), mul(R[5], v.y)), mul(R[8], v.z)), C[2])};
}

// Pose::to_camera: rotation * (x - center) (geometry.hpp:50-51).
__device__ __forceinline__ D3 to_camera(const double* R, const double* C, D3 x) {
    using namespace dev;
    const D3 d{sub(x.x, C[0]), sub(x.y, C[1]), sub(x.z, C[2])};
    return {add(add(mul(R[0], d.x), mul(R[1], d.y)), mul(R[2], d.z)),
            add(add(mul(R[3], d.x), mul(R[4], d.y)), mul(R[5], d.z)),
            add(add(mul(R[6], d.x), mul(R[7], d.y)), mul(R[8], d.z))};
}

// bilinear() of raster.hpp:71-84 on a float raster.
__device__ __forceinline__ double bilinear_f(const float* img, int w, int h, double x, double y) {
    using namespace dev;
    const double xm = double(w - 1), ym = double(h - 1);
    x = x < 0.0 ? 0.0 : (xm < x ? xm : x);
    y = y < 0.0 ? 0.0 : (ym < y ? ym : y);
    const int x0 = static_cast<int>(x), y0 = static_cast<int>(y);
    const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
    const double ax = sub(x, double(x0)), ay = sub(y, double(y0));
    const double top = add(mul(sub(1.0, ax), double(img[y0 * w + x0])), mul(ax, double(img[y0 * w + x1])));
    const double bot = add(mul(sub(1.0, ax), double(img[y1 * w + x0])), mul(ax, double(img[y1 * w + x1])));
    return add(mul(sub(1.0, ay), top), mul(ay, bot));
}

// geometric_consistency_mask (postfilter.cpp:95-160), thread per pixel.
__global__ void geometric_kernel(GeomArgs a) {
    using namespace dev;
    const GeomView& rv = a.views[a.ref];
    const int w = rv.w, h = rv.h;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h)
        return;
    const size_t p = static_cast<size_t>(y) * w + x;
    uint8_t keep = 1;
    const float d = rv.depth[p];
    if (depth_ok(d)) {
        const double xd = double(x), yd = double(y);
        const D3 ray = unproject(rv.k, xd, yd);
        const double dd = double(d);
        const D3 world = to_world(rv.R, rv.C, D3{mul(dd, ray.x), mul(dd, ray.y), mul(dd, ray.z)});
        int hits = 0;
        for (int k = 0; k < a.n; ++k) {
            if (k == a.ref)
                continue;
            const GeomView& nb = a.views[k];
            const D3 cam = to_camera(nb.R, nb.C, world);
            if (cam.z <= 0.0)
                continue;
            const double qx = add(div(mul(nb.k.fx, cam.x), cam.z), nb.k.cx);
            const double qy = add(div(mul(nb.k.fy, cam.y), cam.z), nb.k.cy);
            if (qx < 0.0 || qy < 0.0 || qx > double(nb.w) - 1.0 || qy > double(nb.h) - 1.0)
                continue;
            const int ix = static_cast<int>(lround(qx)), iy = static_cast<int>(lround(qy));
            double dq;
            if (a.bilinear) {
                const int x0 = static_cast<int>(qx), y0 = static_cast<int>(qy);
                const int x1 = min(x0 + 1, nb.w - 1), y1 = min(y0 + 1, nb.h - 1);
                if (depth_ok(nb.depth[y0 * nb.w + x0]) && depth_ok(nb.depth[y0 * nb.w + x1]) &&
                    depth_ok(nb.depth[y1 * nb.w + x0]) && depth_ok(nb.depth[y1 * nb.w + x1]))
                    dq = bilinear_f(nb.depth, nb.w, nb.h, qx, qy);
                else
                    dq = double(nb.depth[iy * nb.w + ix]);
            } else {
                dq = double(nb.depth[iy * nb.w + ix]);
            }
            if (!depth_ok(__double2float_rn(dq)))
                continue;
            const D3 rq = unproject(nb.k, qx, qy);
            const D3 back = to_world(nb.R, nb.C, D3{mul(dq, rq.x), mul(dq, rq.y), mul(dq, rq.z)});
            const D3 rc = to_camera(rv.R, rv.C, back);
            if (rc.z <= 0.0)
                continue;
            const double rx = add(div(mul(rv.k.fx, rc.x), rc.z), rv.k.cx);
            const double ry = add(div(mul(rv.k.fy, rc.y), rc.z), rv.k.cy);
            const double ex = sub(rx, xd), ey = sub(ry, yd);
            if (sqrt_(add(mul(ex, ex), mul(ey, ey))) < a.eta_r)
                ++hits;
        }
        if (hits < a.eta_h)
            keep = 0;
    }
    a.keep[p] = keep;
}

}  // namespace

void gaussian_blur_dog(const uint8_t* img, int w, int h, const BlurKernel& k, float* tmp,
                       uint8_t* mask, cudaStream_t s) {
    blur_rows_kernel<<<grid2(w, h), dim3(32, 8), 0, s>>>(img, w, h, k, tmp);
    blur_cols_dog_kernel<<<grid2(w, h), dim3(32, 8), 0, s>>>(tmp, img, w, h, k, mask);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void gaussian_blur(const uint8_t* img, int w, int h, const BlurKernel& k, float* tmp, float* out,
                   cudaStream_t s) {
    blur_rows_kernel<<<grid2(w, h), dim3(32, 8), 0, s>>>(img, w, h, k, tmp);
    blur_cols_kernel<<<grid2(w, h), dim3(32, 8), 0, s>>>(tmp, w, h, k, out);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void census_transform(const uint8_t* img, int w, int h, int ww, int wh, uint64_t* out, cudaStream_t s) {
    census_kernel<<<grid2(w, h), dim3(32, 8), 0, s>>>(img, w, h, ww, wh, out);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void remove_speckles(uint8_t* mask, int w, int h, uint8_t value, int min_size, int* labels,
                     int* sizes, cudaStream_t s) {
    const dim3 g = grid2(w, h), b(32, 8);
    ccl_init_kernel<<<g, b, 0, s>>>(mask, w, h, value, labels, sizes);
    ccl_merge_kernel<<<g, b, 0, s>>>(mask, w, h, value, labels);
    ccl_count_kernel<<<g, b, 0, s>>>(w, h, labels, sizes);
    ccl_flip_kernel<<<g, b, 0, s>>>(mask, w, h, value, labels, sizes, min_size);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void dilate3(const uint8_t* in, int w, int h, uint8_t* out, cudaStream_t s) {
    dilate3_kernel<<<grid2(w, h), dim3(32, 8), 0, s>>>(in, w, h, out);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void apply_mask(float* depth, float* normals_xyz, float* conf, const uint8_t* mask, int n,
                cudaStream_t s) {
    if (n <= 0)
        return;
    apply_mask_kernel<<<(n + 255) / 256, 256, 0, s>>>(depth, normals_xyz, conf, mask, n);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void geometric_mask(const GeomArgs& a, int w, int h, cudaStream_t s) {
    geometric_kernel<<<grid2(w, h), dim3(32, 8), 0, s>>>(a);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

}  // namespace k
}  // namespace fmvs
