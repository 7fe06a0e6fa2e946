// Accuracy scoring on the device: l1_metrics,
// acc_cpl_f and roc_curve of evaluation.cpp:28-124.
//
// * Counts (valid_est, valid_gt, valid_both, ratio passes per theta) are
//   integer reductions: exact. The ratio test keeps the reference's float ->
//   double expression (evaluation.cpp:22-25).
// * The L1 sums are FP64 reductions in a fixed tree order (per-block shared
//   memory tree, then the block partials summed in block order by one
//   thread): deterministic run to run, equal to the reference's sequential
//   raster-order sum up to FP64 rounding (|rel. diff| ~1e-15).
// * roc_curve: the entries are ordered by descending confidence with ties in
//   raster order by a stable radix sort (CUB) of the confidence keys; the 20
//   prefix pass counts are then exact integer counts, so the error rates are
//   bit-identical to the reference's.
// HBM-bound: 8-12 B read per pixel (+ the sort for the ROC curve).
#include <cub/device/device_radix_sort.cuh>

#include "host.hpp"
#include "kernels.hpp"

namespace fmvs {
namespace k {

namespace {

constexpr int kEvalThreads = 256;

__device__ __forceinline__ bool ratio_pass(float e, float g, double theta) {  // evaluation.cpp:22-25
    using namespace dev;
    const double r = e > g ? div(double(e), double(g)) : div(double(g), double(e));
    return r < theta;
}

__global__ void eval_kernel(const float* __restrict__ est, const float* __restrict__ gt, int n,
                            EvalThetas th, unsigned long long* __restrict__ counts,
                            double* __restrict__ partials) {
    using namespace dev;
    __shared__ double s_abs[kEvalThreads], s_rel[kEvalThreads];
    const int p = blockIdx.x * kEvalThreads + threadIdx.x;
    double dabs = 0.0, drel = 0.0;
    unsigned ev = 0, gv = 0, both = 0;
    unsigned pass_mask = 0;
    if (p < n) {
        const float e = est[p], g = gt[p];
        ev = depth_ok(e);
        gv = depth_ok(g);
        if (ev && gv) {
            both = 1;
            dabs = fabs(sub(double(e), double(g)));  // evaluation.cpp:39-41
            drel = div(dabs, double(g));
            for (int t = 0; t < th.n; ++t)
                if (ratio_pass(e, g, th.theta[t]))
                    pass_mask |= 1u << t;
        }
    }
    // integer counts: warp aggregation + one atomic per warp
    const unsigned full = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const unsigned c_ev = __popc(__ballot_sync(full, ev));
    const unsigned c_gv = __popc(__ballot_sync(full, gv));
    const unsigned c_both = __popc(__ballot_sync(full, both));
    if (lane == 0) {
        atomicAdd(counts + 0, static_cast<unsigned long long>(c_ev));
        atomicAdd(counts + 1, static_cast<unsigned long long>(c_gv));
        atomicAdd(counts + 2, static_cast<unsigned long long>(c_both));
    }
    for (int t = 0; t < th.n; ++t) {
        const unsigned c = __popc(__ballot_sync(full, (pass_mask >> t) & 1u));
        if (lane == 0 && c)
            atomicAdd(counts + 3 + t, static_cast<unsigned long long>(c));
    }
    // FP64 sums: fixed-order tree per block
    s_abs[threadIdx.x] = dabs;
    s_rel[threadIdx.x] = drel;
    __syncthreads();
    for (int o = kEvalThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            s_abs[threadIdx.x] = add(s_abs[threadIdx.x], s_abs[threadIdx.x + o]);
            s_rel[threadIdx.x] = add(s_rel[threadIdx.x], s_rel[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = s_abs[0];
        partials[2 * blockIdx.x + 1] = s_rel[0];
    }
}

__global__ void sum_partials_kernel(const double* __restrict__ partials, int nb, double* out) {
    using namespace dev;
    double a = 0.0, r = 0.0;
    for (int b = 0; b < nb; ++b) {
        a = add(a, partials[2 * b]);
        r = add(r, partials[2 * b + 1]);
    }
    out[0] = a;
    out[1] = r;
}

// ROC entries: key = confidence of each valid estimate (-0 normalised to +0 so
// the sort's ties match the reference comparator), value = ratio pass flag.
__global__ void roc_entries_kernel(const float* __restrict__ est, const float* __restrict__ gt,
                                   const float* __restrict__ conf, int n, double theta,
                                   float* __restrict__ keys, uint8_t* __restrict__ pass,
                                   unsigned long long* __restrict__ count) {
    using namespace dev;
    const int p = blockIdx.x * kEvalThreads + threadIdx.x;
    const bool valid = p < n && depth_ok(est[p]);
    // compaction in raster order: block-local ballot prefix + one atomic per
    // block would reorder blocks, so every pixel keeps its raster slot and
    // invalid ones sort behind all valid keys (key -inf, pass 0)
    if (p < n) {
        keys[p] = valid ? __fadd_rn(conf[p], 0.0f) : -INFINITY;
        pass[p] = valid && depth_ok(gt[p]) && ratio_pass(est[p], gt[p], theta);
    }
    const unsigned c = __popc(__ballot_sync(0xFFFFFFFFu, valid));
    if ((threadIdx.x & 31) == 0 && c)
        atomicAdd(count, static_cast<unsigned long long>(c));
}

__global__ void roc_prefix_kernel(const uint8_t* __restrict__ pass_sorted, int n, RocSteps steps,
                                  unsigned long long* __restrict__ prefix) {
    const int p = blockIdx.x * kEvalThreads + threadIdx.x;
    const bool ps = p < n && pass_sorted[p];
    for (int k = 0; k < 20; ++k) {
        const unsigned c = __popc(__ballot_sync(0xFFFFFFFFu, ps && p < steps.m[k]));
        if ((threadIdx.x & 31) == 0 && c)
            atomicAdd(prefix + k, static_cast<unsigned long long>(c));
    }
}

}  // namespace

void evaluate_counts(const float* est, const float* gt, int n, const EvalThetas& th,
                     unsigned long long* counts, double* partials, double* sums, cudaStream_t s) {
    const int nb = (n + kEvalThreads - 1) / kEvalThreads;
    FMVS_CUDA_CHECK(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * (3 + th.n), s));
    if (nb > 0) {
        eval_kernel<<<nb, kEvalThreads, 0, s>>>(est, gt, n, th, counts, partials);
        sum_partials_kernel<<<1, 1, 0, s>>>(partials, nb, sums);
    }
    FMVS_CUDA_CHECK(cudaGetLastError());
}

size_t roc_scratch_bytes(int n) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, temp, static_cast<const float*>(nullptr),
                                              static_cast<float*>(nullptr),
                                              static_cast<const uint8_t*>(nullptr),
                                              static_cast<uint8_t*>(nullptr), n);
    return temp + 256;
}

void roc_entries(const float* est, const float* gt, const float* conf, int n, double theta,
                 float* keys, uint8_t* pass, unsigned long long* count, cudaStream_t s) {
    FMVS_CUDA_CHECK(cudaMemsetAsync(count, 0, sizeof(unsigned long long), s));
    if (n > 0)
        roc_entries_kernel<<<(n + kEvalThreads - 1) / kEvalThreads, kEvalThreads, 0, s>>>(
            est, gt, conf, n, theta, keys, pass, count);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

void roc_sort_prefix(const float* keys, float* keys_sorted, const uint8_t* pass, uint8_t* pass_sorted,
                     int n, void* temp, size_t temp_bytes, const RocSteps& steps,
                     unsigned long long* prefix, cudaStream_t s) {
    // stable: equal confidences keep raster order (the reference's tie break)
    FMVS_CUDA_CHECK(cub::DeviceRadixSort::SortPairsDescending(temp, temp_bytes, keys, keys_sorted, pass,
                                                              pass_sorted, n, 0, 32, s));
    FMVS_CUDA_CHECK(cudaMemsetAsync(prefix, 0, sizeof(unsigned long long) * 20, s));
    roc_prefix_kernel<<<(n + kEvalThreads - 1) / kEvalThreads, kEvalThreads, 0, s>>>(pass_sorted, n, steps,
                                                                                       prefix);
    FMVS_CUDA_CHECK(cudaGetLastError());
}

}  // namespace k
}  // namespace fmvs
