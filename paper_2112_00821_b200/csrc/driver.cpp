// Host driver and C ABI (include/fmvs.h) of the B200 FaSS-MVS library.
//
// estimate_bundle (pipeline.cpp:200-309) is split into
//   1. a host plan: validation in the reference's order and every
//      data-independent quantity for ALL levels (plane stacks, homographies,
//      lookup tables), uploaded in one H2D copy;
//   2. a fixed device launch sequence on the context stream: pyramid, then per
//      level range -> scan -> sweep -> [SN offsets] -> SGM -> WTA/depth ->
//      median -> normals/smoothing/confidence. The ragged cost volume lives in
//      worst-case arenas, so the sequence never synchronises with the host.
// The stage entry points (fmvs_sweep_cost_volume, fmvs_aggregate, ...) run the
// same kernels on host-provided inputs for stage-wise parity tests.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>
#include <zlib.h>

#include "host.hpp"
#include "kernels.hpp"

namespace k = fmvs::k;
using fmvs::Error;

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return FMVS_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return FMVS_ERR_CUDA;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return FMVS_ERR_CUDA;
    }
}

// Grow-only device buffer.
struct DevBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (ptr)
                cudaFree(ptr);
            ptr = nullptr;
            cap = 0;
            const size_t want = std::max<size_t>(bytes, 256);
            FMVS_CUDA_CHECK(cudaMalloc(&ptr, want));
            cap = want;
        }
        return ptr;
    }
    template <typename T>
    T* as(size_t count) {
        return static_cast<T*>(get(count * sizeof(T)));
    }
    ~DevBuf() {
        if (ptr)
            cudaFree(ptr);
    }
};

// Grow-only pinned host buffer.
struct HostBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (ptr)
                cudaFreeHost(ptr);
            ptr = nullptr;
            cap = 0;
            FMVS_CUDA_CHECK(cudaMallocHost(&ptr, std::max<size_t>(bytes, 256)));
            cap = std::max<size_t>(bytes, 256);
        }
        return ptr;
    }
    ~HostBuf() {
        if (ptr)
            cudaFreeHost(ptr);
    }
};

// Scratch device memory for the stage API (freed on scope exit).
// Stage-API temporaries: stream-ordered allocations from the device's
// memory pool (kept across calls: cudaMemPoolAttrReleaseThreshold is raised
// when a context is created), so a small stage call costs no cudaMalloc /
// cudaFree round trips -- the reference's acceptance criterion 1 times 1800
// of them against a 10 s budget.
struct Tmp {
    explicit Tmp(cudaStream_t stream) : s(stream) {}
    cudaStream_t s;
    std::vector<void*> ptrs;
    template <typename T>
    T* alloc(size_t count) {
        void* p = nullptr;
        // + 256 B: kernels may over-read a volume's tail by up to a 48-byte
        // aligned chunk (SGM cost staging) or add 0 past it (SGM REDs)
        FMVS_CUDA_CHECK(cudaMallocAsync(&p, count * sizeof(T) + 256, s));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    template <typename T>
    T* upload(const T* host, size_t count, cudaStream_t s) {
        T* d = alloc<T>(count);
        if (count)
            FMVS_CUDA_CHECK(cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
        return d;
    }
    ~Tmp() {
        for (void* p : ptrs)
            cudaFreeAsync(p, s);
    }
};

fmvs::V3 v3(const double* n) { return {n[0], n[1], n[2]}; }

// Lane blocking of the SGM kernel at the refined levels: G lanes per scanline,
// K hypotheses per lane and pass (FMVS_SGM_G / FMVS_SGM_K; results are
// identical, only speed differs). G = 0 selects the one-line-per-warp kernel.
// Lanes per scanline and hypotheses per lane of the refined-level SGM.
// `widest` bounds the pixels' hypothesis counts when known (0: unknown): the
// default spacing-multiple policy (3 coarser spacings) gives <= 12, one
// G=4 x K=3 pass; wider pixels take the kernel's multi-pass lines.
void sgm_blocking(int* g, int* k, int widest = 0) {
    *g = 4;
    *k = widest > 0 && widest <= 12 ? 3 : 4;
    if (const char* e = std::getenv("FMVS_SGM_G"))
        *g = std::atoi(e);
    if (const char* e = std::getenv("FMVS_SGM_K"))
        *k = std::atoi(e);
}

// Per-context budget of cost-volume entries for worst-case arenas
// (FMVS_ARENA_ENTRIES overrides; default 2^30 entries = 6 GB of costs +
// aggregate, which covers Full-HD at 511 planes).
size_t arena_budget_entries() {
    if (const char* e = std::getenv("FMVS_ARENA_ENTRIES"))
        return static_cast<size_t>(std::strtoull(e, nullptr, 10));
    return size_t(1) << 30;
}

fmvs::dev::Intr intr_of(const fmvs_intrinsics& k) { return fmvs::dev::make_intr(k); }

// Host plan of one level (everything data-independent).
struct LevelPlan {
    int w = 0, h = 0;
    std::vector<fmvs_intrinsics> intr;  // per view
    std::vector<double> planes;
    std::vector<double> homs;           // [nmatch][P][9]
    // offsets into the uploaded plan blob (in doubles)
    size_t off_planes = 0, off_homs = 0;
    size_t off_ux = 0, off_uy = 0;      // the reference view's unprojection tables
    size_t img_off = 0;                 // per-level byte offset of the image block
    size_t quad_off = 0;                // per-level u32 offset of the quad block
};

// Validation + geometry for a whole bundle (pipeline.cpp:202-242,
// matching.cpp:119-142), evaluated before any launch.
std::vector<LevelPlan> plan_bundle(const fmvs_view* views, int n, const fmvs_config& cfg) {
    fmvs::validate_config(cfg);
    if (n < 3 || n % 2 == 0)
        fmvs::fail_input("estimate: bundle must hold an odd number (>= 3) of views");
    if (!views)
        fmvs::fail_input("estimate: no views");
    for (int i = 0; i < n; ++i)
        fmvs::validate_view(views[i]);
    const int ref = n / 2;
    const int L = cfg.pyramid_levels;
    const fmvs::V3 normal = v3(cfg.sweep_normal);

    std::vector<LevelPlan> lv(L);
    for (int l = 0; l < L; ++l) {
        lv[l].intr.resize(n);
        for (int k = 0; k < n; ++k)
            lv[l].intr[k] = l == 0 ? views[k].intrinsics : fmvs::halved(lv[l - 1].intr[k]);
        lv[l].w = lv[l].intr[ref].width;
        lv[l].h = lv[l].intr[ref].height;
    }
    for (int l = L - 1; l >= 0; --l) {
        LevelPlan& P = lv[l];
        std::vector<fmvs::Camera> cams(n);
        for (int k = 0; k < n; ++k)
            cams[k] = fmvs::camera_of(P.intr[k], views[k].pose);
        double dmin = 0, dmax = 0;
        fmvs::bounding_distances(cfg.d_min, cfg.d_max, normal, P.intr[ref], &dmin, &dmax);
        int far_view = ref == 0 ? 1 : 0;
        double far_dist = -1.0;
        for (int k = 0; k < n; ++k) {
            if (k == ref)
                continue;
            const double dist = fmvs::norm(fmvs::sub(cams[k].center, cams[ref].center));
            if (dist > far_dist) {
                far_dist = dist;
                far_view = k;
            }
        }
        const int cap = l == L - 1 ? cfg.max_planes : std::numeric_limits<int>::max();
        P.planes = fmvs::plane_distances(cams[ref], cams[far_view], dmin, dmax, normal, cap);
        if (l < L - 1 && cfg.range_kind == FMVS_RANGE_SPACING_MULTIPLE && lv[l + 1].planes.size() < 2)
            fmvs::fail_config("refine range: spacing policy needs the coarser plane stack");
        if (P.planes.size() > 65535)
            fmvs::fail_config("b200: more than 65535 sweep planes in one level is unsupported");
        // sweep_cost_volume checks (matching.cpp:126-142)
        for (size_t i = 1; i < P.planes.size(); ++i)
            if (!(P.planes[i] < P.planes[i - 1]))
                fmvs::fail_input("sweep: plane distances must be strictly decreasing");
        std::vector<fmvs::V3> centers;
        for (int k = 0; k < n; ++k)
            centers.push_back(fmvs::mul(cams[ref].rot, fmvs::sub(cams[k].center, cams[ref].center)));
        fmvs::require_centers_in_front(normal, P.planes.back(), centers);
        const int np = static_cast<int>(P.planes.size());
        P.homs.resize(static_cast<size_t>(n - 1) * np * 9);
        int m = 0;
        for (int k = 0; k < n; ++k) {
            if (k == ref)
                continue;
            for (int i = 0; i < np; ++i) {
                const fmvs::M3 H = fmvs::plane_homography(normal, P.planes[i], cams[ref], cams[k]);
                double* o = &P.homs[(static_cast<size_t>(m) * np + i) * 9];
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c)
                        o[3 * r + c] = H.a[r][c];
            }
            ++m;
        }
    }
    fmvs_sgm_config sc = cfg.sgm;
    sc.penalty_scale = n / 2;
    fmvs::validate_sgm(sc);
    return lv;
}

}  // namespace

struct fmvs_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t staged = nullptr;   // plan upload finished reading the pinned blob
    HostBuf pinned_plan;
    HostBuf pinned_stats;
    std::map<std::string, std::unique_ptr<DevBuf>> bufs;
    std::vector<fmvs_level_stats> stats;
    int64_t launches = 0;
    // optional per-stage CUDA-event timing (bench.py roofline numbers)
    bool timing = false;
    int sweep_exact = 0;  // FMVS_SWEEP_EXACT=1: force the exact per-hypothesis sweep
    int sweep_stats = 0;  // FMVS_SWEEP_STATS=1 (2 + l: level l only): count certified-census fallbacks
    bool agg16 = true;    // packed u16 SGM aggregate where provably exact (FMVS_SGM_AGG16=0: off)
    uint64_t agg16_min = uint64_t(48) << 20;  // ... on uniform levels above this many entries
                                              // (FMVS_SGM_AGG16_MIN: test hook)
    // stage capture of one level (fmvs_ctx_set_capture)
    struct Capture {
        int level = -1;
        int w = 0, h = 0;
        std::vector<fmvs::dev::VolMeta> meta;
        std::vector<uint64_t> row_base;
        std::vector<uint16_t> costs;
        std::vector<uint32_t> agg;
        std::vector<int32_t> winners;
        std::vector<float> depth_raw;
    } cap;
    struct Span {
        int stage;
        cudaEvent_t a, b;
    };
    std::vector<Span> spans;
    std::vector<cudaEvent_t> event_pool;
    std::vector<std::string> stage_names;
    std::vector<double> stage_ms;
    std::vector<int64_t> stage_calls;

    cudaEvent_t event() {
        if (!event_pool.empty()) {
            cudaEvent_t e = event_pool.back();
            event_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        FMVS_CUDA_CHECK(cudaEventCreate(&e));
        return e;
    }
    int stage_id(const char* name) {
        for (size_t i = 0; i < stage_names.size(); ++i)
            if (stage_names[i] == name)
                return static_cast<int>(i);
        stage_names.push_back(name);
        stage_ms.push_back(0.0);
        stage_calls.push_back(0);
        return static_cast<int>(stage_names.size() - 1);
    }
    // Runs launch() bracketed by events on the context stream when timing.
    template <typename F>
    void timed(const char* name, F&& launch) {
        if (!timing) {
            launch();
            return;
        }
        Span sp{stage_id(name), event(), event()};
        FMVS_CUDA_CHECK(cudaEventRecord(sp.a, stream));
        launch();
        FMVS_CUDA_CHECK(cudaEventRecord(sp.b, stream));
        spans.push_back(sp);
    }
    // After a stream synchronisation: fold finished spans into the totals.
    void collect() {
        for (const Span& sp : spans) {
            float ms = 0.0f;
            FMVS_CUDA_CHECK(cudaEventElapsedTime(&ms, sp.a, sp.b));
            stage_ms[sp.stage] += ms;
            stage_calls[sp.stage] += 1;
            event_pool.push_back(sp.a);
            event_pool.push_back(sp.b);
        }
        spans.clear();
    }

    DevBuf& buf(const std::string& name) {
        auto& b = bufs[name];
        if (!b)
            b = std::make_unique<DevBuf>();
        return *b;
    }
    void use() { FMVS_CUDA_CHECK(cudaSetDevice(device)); }
};

namespace {

// The per-bundle device pipeline. d_images[k] are level-0 device images;
// outputs are device pointers of the reference view's level-0 maps.
void run_bundle(fmvs_ctx* ctx, const fmvs_view* views, int n, const fmvs_config& cfg,
                const uint8_t* const* d_images, float* d_depth, float* d_normals, float* d_conf) {
    std::vector<LevelPlan> lv = plan_bundle(views, n, cfg);
    const int L = cfg.pyramid_levels;
    const int ref = n / 2;
    const int nmatch = n - 1;
    cudaStream_t s = ctx->stream;
    int64_t launches = 0;

    // ---- plan blob: per level planes + homs, LUTs, quad pointers ----------
    const fmvs_sgm_config sgm_base = cfg.sgm;
    fmvs_sgm_config sc = sgm_base;
    sc.penalty_scale = n / 2;  // pipeline.cpp:252-253
    const std::vector<long long> phi2 = fmvs::phi2_table(sc);
    const int census_bits = cfg.cost.window_w * cfg.cost.window_h - 1;
    const std::vector<uint16_t> clut = fmvs::census_cost_table(census_bits);
    const std::vector<double> swt = fmvs::smoothing_table(cfg.normal_smoothing_radius);
    double k3[3];
    fmvs::blur3_kernel(k3);

    size_t nd = 0;  // doubles
    for (auto& P : lv) {
        P.off_planes = nd;
        nd += P.planes.size();
        P.off_homs = nd;
        nd += P.homs.size();
        P.off_ux = nd;
        nd += static_cast<size_t>(P.intr[ref].width) + 2;
        P.off_uy = nd;
        nd += static_cast<size_t>(P.intr[ref].height) + 2;
    }
    const size_t off_swt = nd;
    nd += swt.size();
    const size_t off_phi2 = nd;  // long long, same width as double
    nd += 256;
    size_t img_bytes = 0, quad_words = 0;
    for (auto& P : lv) {
        P.img_off = img_bytes;
        P.quad_off = quad_words;
        size_t px = 0;
        for (int k2 = 0; k2 < n; ++k2)
            px += static_cast<size_t>(P.intr[k2].width) * P.intr[k2].height;
        img_bytes += px;
        quad_words += px;
    }
    const size_t off_ptrs = nd;  // quad pointers (per level, nmatch), as 8-byte words
    nd += static_cast<size_t>(L) * nmatch;
    const size_t off_sizes = nd;  // int2 per level/match (8 bytes)
    nd += static_cast<size_t>(L) * nmatch;
    const size_t off_clut = nd;
    nd += (clut.size() * 2 + 7) / 8;

    double* d_blob = ctx->buf("plan").as<double>(nd);
    uint8_t* d_img = ctx->buf("images").as<uint8_t>(img_bytes);
    uint32_t* d_quad = ctx->buf("quads").as<uint32_t>(quad_words);

    FMVS_CUDA_CHECK(cudaEventSynchronize(ctx->staged));
    double* h_blob = static_cast<double*>(ctx->pinned_plan.get(nd * sizeof(double)));
    for (auto& P : lv) {
        std::memcpy(h_blob + P.off_planes, P.planes.data(), P.planes.size() * 8);
        std::memcpy(h_blob + P.off_homs, P.homs.data(), P.homs.size() * 8);
        // unproject's divisions (geometry.hpp:28-30), x / y in [-1, size]
        const fmvs_intrinsics& k = P.intr[ref];
        for (int x = -1; x <= k.width; ++x)
            h_blob[P.off_ux + x + 1] = (double(x) - k.cx) / k.fx;
        for (int y = -1; y <= k.height; ++y)
            h_blob[P.off_uy + y + 1] = (double(y) - k.cy) / k.fy;
    }
    std::memcpy(h_blob + off_swt, swt.data(), swt.size() * 8);
    std::memcpy(h_blob + off_phi2, phi2.data(), 256 * 8);
    std::memcpy(h_blob + off_clut, clut.data(), clut.size() * 2);
    std::vector<const uint8_t*> img_ptr(static_cast<size_t>(L) * n);
    for (int l = 0; l < L; ++l) {
        size_t o = lv[l].img_off, q = lv[l].quad_off;
        int m = 0;
        for (int k2 = 0; k2 < n; ++k2) {
            const size_t px = static_cast<size_t>(lv[l].intr[k2].width) * lv[l].intr[k2].height;
            img_ptr[l * n + k2] = l == 0 ? d_images[k2] : d_img + o;
            if (k2 != ref) {
                const uint32_t* qp = d_quad + q;
                std::memcpy(h_blob + off_ptrs + l * nmatch + m, &qp, 8);
                const int2 sz = make_int2(lv[l].intr[k2].width, lv[l].intr[k2].height);
                std::memcpy(h_blob + off_sizes + l * nmatch + m, &sz, 8);
                ++m;
            }
            o += px;
            q += px;
        }
    }
    FMVS_CUDA_CHECK(cudaMemcpyAsync(d_blob, h_blob, nd * sizeof(double), cudaMemcpyHostToDevice, s));
    FMVS_CUDA_CHECK(cudaEventRecord(ctx->staged, s));
    const long long* d_phi2 = reinterpret_cast<const long long*>(d_blob + off_phi2);
    const double* d_swt = d_blob + off_swt;
    const uint16_t* d_clut = reinterpret_cast<const uint16_t*>(d_blob + off_clut);

    // ---- K1: pyramid + quads (one launch per pyramid level, one per quad
    // batch: blockIdx.z selects the view) ------------------------------------
    for (int l = 1; l < L; ++l)
        for (int k0 = 0; k0 < n; k0 += k::kImgBatch) {
            k::ImgBatch b{};
            const int m = std::min(n - k0, k::kImgBatch);
            for (int i = 0; i < m; ++i) {
                const fmvs_intrinsics& a = lv[l - 1].intr[k0 + i];
                const fmvs_intrinsics& c = lv[l].intr[k0 + i];
                b.job[i] = k::ImgJob{img_ptr[(l - 1) * n + k0 + i], const_cast<uint8_t*>(img_ptr[l * n + k0 + i]),
                                     nullptr, a.width, a.height, c.width, c.height};
            }
            ctx->timed("pyramid", [&] { k::blur_halve_batch(b, m, k3, s); });
            ++launches;
        }
    {
        k::ImgBatch b{};
        int m = 0;
        auto flush = [&] {
            if (m == 0)
                return;
            ctx->timed("quads", [&] { k::pack_quads_batch(b, m, s); });
            ++launches;
            m = 0;
        };
        for (int l = 0; l < L; ++l) {
            size_t q = lv[l].quad_off;
            for (int k2 = 0; k2 < n; ++k2) {
                const fmvs_intrinsics& a = lv[l].intr[k2];
                if (k2 != ref) {
                    b.job[m++] = k::ImgJob{img_ptr[l * n + k2], nullptr, d_quad + q, a.width, a.height, 0, 0};
                    if (m == k::kImgBatch)
                        flush();
                }
                q += static_cast<size_t>(a.width) * a.height;
            }
        }
        flush();
    }

    // ---- per-level buffers ---------------------------------------------------
    size_t max_px = 0, max_entries = 0;
    int max_h = 0, max_p = 0;
    for (auto& P : lv) {
        const size_t px = static_cast<size_t>(P.w) * P.h;
        max_px = std::max(max_px, px);
        max_entries = std::max(max_entries, px * P.planes.size());
        max_h = std::max(max_h, P.h);
        max_p = std::max(max_p, static_cast<int>(P.planes.size()));
    }
    auto* meta = ctx->buf("meta").as<fmvs::dev::VolMeta>(max_px);
    auto* row_total = ctx->buf("row_total").as<uint32_t>(max_h);
    auto* row_base = ctx->buf("row_base").as<uint64_t>(static_cast<size_t>(L) * (max_h + 1));
    // Cost-volume arenas (u16 costs + u32 aggregate). Worst case W*H*P per
    // level, allocated once, keeps the whole bundle one asynchronous launch
    // sequence. When that exceeds the per-context budget (4K inputs: 51 GB),
    // each level is sized to its actual entry count instead: one host
    // synchronisation after the level's range kernels.
    const size_t arena_budget = arena_budget_entries();
    const bool compact = max_entries > arena_budget;
    uint16_t* costs = nullptr;
    uint32_t* agg = nullptr;
    if (!compact) {
        costs = ctx->buf("costs").as<uint16_t>(max_entries + k::kAggSlack);
        agg = ctx->buf("agg").as<uint32_t>(max_entries + k::kAggSlack);
    }
    auto* offs = ctx->buf("offsets").as<int16_t>(4 * max_px);
    auto* depth_raw = ctx->buf("depth_raw").as<float>(max_px);
    auto* nraw = ctx->buf("normals_raw").as<float>(3 * max_px);
    size_t lvl_px = 0;
    for (auto& P : lv)
        lvl_px += static_cast<size_t>(P.w) * P.h;
    float* depth_all = ctx->buf("depth_levels").as<float>(lvl_px);
    float* normals_all = ctx->buf("normal_levels").as<float>(3 * lvl_px);
    std::vector<float*> depth_l(L), normals_l(L);
    {
        size_t o = 0;
        for (int l = 0; l < L; ++l) {
            depth_l[l] = depth_all + o;
            normals_l[l] = normals_all + 3 * o;
            o += static_cast<size_t>(lv[l].w) * lv[l].h;
        }
        depth_l[0] = d_depth;
        normals_l[0] = d_normals;
    }
    int pmax_smem_limit = (200 * 1024) / (4 * 2 * 4);
    uint32_t* sgm_scratch = nullptr;
    {
        size_t lines = 0;
        for (auto& P : lv)
            lines = std::max(lines, static_cast<size_t>(k::sgm_total_lines(P.w, P.h, 8)));
        sgm_scratch = ctx->buf("sgm_scratch").as<uint32_t>(lines * 2 * (max_p + k::kSgmLinePad));
    }
    uint32_t* sgm_line = ctx->buf("sgm_line").as<uint32_t>(k::sgm_line_scratch_words(lv[0].w, lv[0].h));

    const double cos_rho = std::cos(60.0 * M_PI / 180.0);
    const double pdv = (cfg.sweep_normal[0] * 0.0 + cfg.sweep_normal[1] * 0.0) +
                       cfg.sweep_normal[2] * -1.0;
    const double nx = cfg.sweep_normal[0], ny = cfg.sweep_normal[1], nz = cfg.sweep_normal[2];

    ctx->stats.assign(L, fmvs_level_stats{});
    for (int l = L - 1; l >= 0; --l) {
        const LevelPlan& P = lv[l];
        const int np = static_cast<int>(P.planes.size());
        const double* d_planes = d_blob + P.off_planes;
        fmvs::dev::Intr intr = intr_of(P.intr[ref]);
        intr.ux = d_blob + P.off_ux;
        intr.uy = d_blob + P.off_uy;
        uint64_t* rb = row_base + static_cast<size_t>(l) * (max_h + 1);
        const bool have_prior = l < L - 1;

        k::RangeArgs ra{};
        ra.intr = intr;
        ra.nx = nx;
        ra.ny = ny;
        ra.nz = nz;
        ra.planes = d_planes;
        ra.nplanes = np;
        ra.d_min = cfg.d_min;
        ra.d_max = cfg.d_max;
        ra.mode = have_prior ? 1 : 0;
        if (have_prior) {
            ra.prior = depth_l[l + 1];
            ra.prior_w = lv[l + 1].w;
            ra.prior_h = lv[l + 1].h;
            ra.policy = cfg.range_kind;
            ra.policy_value = cfg.range_value;
            ra.coarser = d_blob + lv[l + 1].off_planes;
            ra.ncoarser = static_cast<int>(lv[l + 1].planes.size());
        }
        ra.meta = meta;
        ra.row_total = row_total;
        ctx->timed("range", [&] {
            k::range_rows(ra, s);
            k::scan_rows(row_total, P.h, rb, s);
        });
        launches += 2;
        uint64_t entries_bound = static_cast<uint64_t>(P.w) * P.h * np;
        if (compact) {
            uint64_t entries = 0;
            FMVS_CUDA_CHECK(cudaMemcpyAsync(&entries, rb + P.h, sizeof(entries), cudaMemcpyDeviceToHost, s));
            FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
            entries_bound = entries;
            const size_t need = std::max<size_t>(entries, 1);
            costs = ctx->buf("costs").as<uint16_t>(need + k::kAggSlack);
            agg = ctx->buf("agg").as<uint32_t>(need + k::kAggSlack);
        }

        k::SweepArgs sa{};
        sa.w = P.w;
        sa.h = P.h;
        sa.ref_img = img_ptr[l * n + ref];
        sa.nmatch = nmatch;
        sa.quads = reinterpret_cast<const uint32_t* const*>(d_blob + off_ptrs + l * nmatch);
        sa.sizes = reinterpret_cast<const int2*>(d_blob + off_sizes + l * nmatch);
        sa.homs = d_blob + P.off_homs;
        sa.nplanes = np;
        sa.nleft = ref;
        sa.meta = meta;
        sa.row_base = rb;
        sa.costs = costs;
        sa.kind = cfg.cost.kind;
        sa.ww = cfg.cost.window_w;
        sa.wh = cfg.cost.window_h;
        sa.census_lut = d_clut;
        sa.disable_tiled = ctx->sweep_exact;
        sa.plane_slicing = l == L - 1;  // uniform ranges: every pixel sweeps the whole stack
        sa.narrow_max = l == L - 1 ? 65535 : 0;
        sa.small_lists = std::getenv("FMVS_NCC_SMALL_LISTS") != nullptr;
        if (ctx->sweep_stats == 1 || ctx->sweep_stats == 2 + l)
            sa.stats = ctx->buf("sweep_stats").as<unsigned long long>(8);
        ctx->timed(l == 0 ? "sweep_l0" : "sweep", [&] { launches += k::sweep(sa, s); });

        int variant = cfg.sgm.variant;
        if (variant == FMVS_SGM_SURFACE_NORMAL && !have_prior)
            variant = FMVS_SGM_PLANE;  // pipeline.cpp:254-255
        if (variant == FMVS_SGM_SURFACE_NORMAL) {
            k::OffsetArgs oa{};
            oa.intr = intr;
            oa.w = P.w;
            oa.h = P.h;
            oa.prior_depth = depth_l[l + 1];
            oa.prior_normals = normals_l[l + 1];
            oa.prior_w = lv[l + 1].w;
            oa.prior_h = lv[l + 1].h;
            oa.nx = nx;
            oa.ny = ny;
            oa.nz = nz;
            oa.planes = d_planes;
            oa.nplanes = np;
            oa.out = offs;
            ctx->timed("offsets", [&] { k::normal_offsets(oa, s); });
            ++launches;
        }

        k::SgmArgs ga{};
        ga.w = P.w;
        ga.h = P.h;
        ga.meta = meta;
        ga.row_base = rb;
        ga.costs = costs;
        ga.agg = agg;
        ga.image = img_ptr[l * n + ref];
        ga.variant = variant;
        ga.phi1 = std::llround(sc.phi1 * sc.penalty_scale);
        ga.phi2_lut = d_phi2;
        ga.phi2_max = *std::max_element(phi2.begin(), phi2.end());
        ga.offsets = variant == FMVS_SGM_SURFACE_NORMAL ? offs : nullptr;
        ga.intr = intr;
        ga.nx = nx;
        ga.ny = ny;
        ga.nz = nz;
        ga.planes = d_planes;
        ga.nplanes = np;
        static const int kDirs[8][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1},
                                        {1, 1}, {-1, -1}, {1, -1}, {-1, 1}};
        ga.ndirs = cfg.sgm.paths == 8 ? 8 : 4;
        for (int d = 0; d < 8; ++d) {
            ga.dirs[d][0] = kDirs[d][0];
            ga.dirs[d][1] = kDirs[d][1];
        }
        ga.pmax = np;
        // coarsest level: dense ranges, one line per warp-wide group; refined
        // levels: ~12 hypotheses per pixel, 32/G lines per warp
        // spacing multiple m: about 4m + 1 finer planes per pixel
        const bool narrow_policy = cfg.range_kind == FMVS_RANGE_SPACING_MULTIPLE && cfg.range_value <= 3.0;
        sgm_blocking(&ga.group, &ga.kper, narrow_policy ? 12 : 0);
        if (l == L - 1) {  // dense coarsest level: one line per warp, one pass up to 256 planes
            ga.group = 32;
            ga.kper = np > 128 ? 8 : 4;
        }
        ga.group_caps = l == L - 1 ? std::min(np, 1024) : 32;
        ga.scratch = (ga.group > 0 || np > pmax_smem_limit) ? sgm_scratch : nullptr;
        ga.line_scratch = sgm_line;
        ga.entries_bound = entries_bound;
        // packed u16 aggregate when every sum provably fits (a view's cost is
        // <= 255: census LUT / NCC truncation / outside; a pixel's the smaller
        // side's sum, matching.cpp:283-292) AND the u32 aggregate would not
        // stay in L2: then each RED misses and costs a DRAM read + write, and
        // halving the bytes wins (C3: SGM 7.35 -> 5.59 ms); an L2-resident
        // aggregate is faster unpacked (two lanes per word serialise their
        // REDs: C2 L0 0.63 -> 0.79 ms; C4 L0, 100 M entries of ~12 per
        // pixel, 2.36 -> 2.61 ms). Only the uniform (coarsest, one line per
        // warp, long contiguous runs) levels qualify: C4 L2 1.8x less DRAM.
        const uint64_t known_entries = have_prior ? 0 : entries_bound;
        ga.cost_max = 255 * std::max(ref, nmatch - ref);
        ga.agg16 = ctx->agg16 && known_entries > ctx->agg16_min && k::sgm_agg16_ok(ga, ga.cost_max);
        // the SGM accumulator of the level (make_accumulator, sgm.cpp:198-208)
        ctx->timed("zero", [&] { k::zero_entries(agg, rb + P.h, s, ga.agg16 != 0); });
        ++launches;
        ctx->timed(l == 0 ? "sgm_l0" : "sgm", [&] { k::sgm(ga, s); });
        ++launches;

        k::WtaArgs wa{};
        wa.w = P.w;
        wa.h = P.h;
        wa.meta = meta;
        wa.row_base = rb;
        wa.agg = agg;
        wa.agg16 = ga.agg16;
        wa.depth = depth_raw;
        wa.intr = intr;
        wa.nx = nx;
        wa.ny = ny;
        wa.nz = nz;
        wa.planes = d_planes;
        wa.nplanes = np;
        wa.wide = !have_prior && np >= 64;  // uniform level: every pixel scans the whole stack
        const bool capture = ctx->cap.level == l;
        if (capture)
            wa.winners = ctx->buf("cap_winners").as<int32_t>(static_cast<size_t>(P.w) * P.h);
        ctx->timed("wta", [&] { k::wta_depth(wa, s); });
        if (capture) {
            // debug path: synchronous copies of the level's intermediates
            auto& c = ctx->cap;
            const size_t px = static_cast<size_t>(P.w) * P.h;
            c.w = P.w;
            c.h = P.h;
            c.meta.resize(px);
            c.row_base.resize(P.h + 1);
            c.winners.resize(px);
            c.depth_raw.resize(px);
            FMVS_CUDA_CHECK(cudaMemcpyAsync(c.meta.data(), meta, px * sizeof(fmvs::dev::VolMeta),
                                            cudaMemcpyDeviceToHost, s));
            FMVS_CUDA_CHECK(cudaMemcpyAsync(c.row_base.data(), rb, (P.h + 1) * 8, cudaMemcpyDeviceToHost, s));
            FMVS_CUDA_CHECK(cudaMemcpyAsync(c.winners.data(), wa.winners, px * 4, cudaMemcpyDeviceToHost, s));
            FMVS_CUDA_CHECK(cudaMemcpyAsync(c.depth_raw.data(), depth_raw, px * 4, cudaMemcpyDeviceToHost, s));
            FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
            const size_t entries = c.row_base[P.h];
            c.costs.resize(entries);
            c.agg.resize(entries);
            FMVS_CUDA_CHECK(cudaMemcpyAsync(c.costs.data(), costs, entries * 2, cudaMemcpyDeviceToHost, s));
            if (ga.agg16) {  // packed u16 aggregate: widen to the reference's u32
                std::vector<uint16_t> a16(entries);
                FMVS_CUDA_CHECK(cudaMemcpyAsync(a16.data(), agg, entries * 2, cudaMemcpyDeviceToHost, s));
                FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
                std::copy(a16.begin(), a16.end(), c.agg.begin());
            } else {
                FMVS_CUDA_CHECK(cudaMemcpyAsync(c.agg.data(), agg, entries * 4, cudaMemcpyDeviceToHost, s));
            }
            FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
            c.level = -1;
        }
        ctx->timed("median", [&] { k::median5(depth_raw, P.w, P.h, depth_l[l], s); });
        launches += 2;

        // Normals are consumed only by SN below level 0 and by the result at
        // level 0 (pipeline.cpp:292-306); confidence only at level 0.
        const bool need_normals = l == 0 || cfg.sgm.variant == FMVS_SGM_SURFACE_NORMAL;
        if (need_normals) {
            ctx->timed("normals", [&] { k::normals_raw(depth_l[l], P.w, P.h, intr, nraw, s); });
            ctx->timed("smooth_conf", [&] {
                k::smooth_conf(nraw, img_ptr[l * n + ref], P.w, P.h, cfg.normal_smoothing_radius,
                               d_swt, normals_l[l], l == 0 ? d_conf : nullptr, cos_rho, pdv, nx, ny,
                               nz, s);
            });
            launches += 2;
        }
        ctx->stats[l] = fmvs_level_stats{P.w, P.h, np, 0};
    }
    // entry totals per level (read back after the caller synchronises)
    auto* h_stats = static_cast<uint64_t*>(ctx->pinned_stats.get(sizeof(uint64_t) * L));
    for (int l = 0; l < L; ++l)
        FMVS_CUDA_CHECK(cudaMemcpyAsync(h_stats + l, row_base + static_cast<size_t>(l) * (max_h + 1) + lv[l].h,
                                        sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    ctx->launches = launches;
}

void finish_stats(fmvs_ctx* ctx) {
    auto* h = static_cast<uint64_t*>(ctx->pinned_stats.ptr);
    if (!h)
        return;
    for (size_t l = 0; l < ctx->stats.size(); ++l)
        ctx->stats[l].entries = h[l];
}

void copy_views_to_device(fmvs_ctx* ctx, const fmvs_view* views, int n,
                          std::vector<const uint8_t*>* d_images) {
    size_t total = 0;
    for (int k2 = 0; k2 < n; ++k2)
        total += static_cast<size_t>(views[k2].intrinsics.width) * views[k2].intrinsics.height;
    uint8_t* d = ctx->buf("input_images").as<uint8_t>(total);
    d_images->resize(n);
    size_t o = 0;
    for (int k2 = 0; k2 < n; ++k2) {
        const size_t px = static_cast<size_t>(views[k2].intrinsics.width) * views[k2].intrinsics.height;
        FMVS_CUDA_CHECK(cudaMemcpyAsync(d + o, views[k2].image, px, cudaMemcpyHostToDevice, ctx->stream));
        (*d_images)[k2] = d + o;
        o += px;
    }
}

// Converts the reference ragged layout (first, count, offset) to meta + row
// bases. The reference allows any per-pixel offsets (matching.hpp:36-53: a
// pixel's entries are costs[offset[p], offset[p] + count[p]); test_sgm.cpp:262
// zeroes a count in place); the device layout is the compact prefix sum, so a
// non-compact input is gathered: *src receives each compact entry's source
// index (empty when the input is already compact). *compact_total = sum of
// counts.
void host_layout(int w, int h, const int32_t* first, const int32_t* count, const uint64_t* offset,
                 uint64_t total, std::vector<fmvs::dev::VolMeta>* meta, std::vector<uint64_t>* rb,
                 std::vector<uint64_t>* src, uint64_t* compact_total) {
    const size_t px = static_cast<size_t>(w) * h;
    meta->resize(px);
    rb->resize(h + 1);
    src->clear();
    bool compact = true;
    uint64_t run = 0;
    for (size_t p = 0; p < px; ++p) {
        if (first[p] < 0 || first[p] > 65535 || count[p] < 0 || count[p] > 65535)
            fmvs::fail_input("b200 layout: first/count out of the supported range");
        if (offset[p] + static_cast<uint64_t>(count[p]) > total)
            fmvs::fail_input("b200 layout: a pixel's entries lie outside the cost array");
        if (count[p] > 0 && offset[p] != run)
            compact = false;
        run += static_cast<uint64_t>(count[p]);
    }
    *compact_total = run;
    if (!compact)
        src->reserve(run);
    run = 0;
    for (int y = 0; y < h; ++y) {
        const size_t row = static_cast<size_t>(y) * w;
        (*rb)[y] = run;
        for (int x = 0; x < w; ++x) {
            const size_t p = row + x;
            (*meta)[p] = fmvs::dev::VolMeta{static_cast<uint32_t>(run - (*rb)[y]),
                                            static_cast<uint32_t>(first[p]) |
                                                (static_cast<uint32_t>(count[p]) << 16)};
            if (!compact)
                for (int32_t i = 0; i < count[p]; ++i)
                    src->push_back(offset[p] + i);
            run += static_cast<uint64_t>(count[p]);
        }
    }
    (*rb)[h] = run;
}

template <typename T>
std::vector<T> gather(const T* in, const std::vector<uint64_t>& src) {
    std::vector<T> out(src.size());
    for (size_t i = 0; i < src.size(); ++i)
        out[i] = in[src[i]];
    return out;
}

}  // namespace

// ======================================================================= ABI

extern "C" {

int32_t fmvs_abi_version(void) { return FMVS_ABI_VERSION; }

const char* fmvs_last_error(void) { return g_last_error.c_str(); }

void fmvs_config_default(fmvs_config* c, double d_min, double d_max) {
    c->bundle_size = 5;
    c->pyramid_levels = 3;
    c->d_min = d_min;
    c->d_max = d_max;
    c->sweep_normal[0] = 0;
    c->sweep_normal[1] = 0;
    c->sweep_normal[2] = -1;
    c->range_kind = FMVS_RANGE_SPACING_MULTIPLE;
    c->range_value = 3.0;
    c->max_planes = 256;
    c->sgm = {FMVS_SGM_PLANE, 8, 100.0, 1, 0.0, 8.0, 10.0, 1};
    c->cost = {FMVS_COST_NCC, 5, 5};
    c->normal_smoothing_radius = 2;
}

int fmvs_ctx_create(int32_t device, fmvs_ctx** out) {
    return guarded([&] {
        if (!out)
            fmvs::fail_input("ctx: null output");
        if (device < 0)
            FMVS_CUDA_CHECK(cudaGetDevice(&device));
        auto ctx = std::make_unique<fmvs_ctx>();
        ctx->device = device;
        if (const char* e = std::getenv("FMVS_SWEEP_EXACT"))
            ctx->sweep_exact = std::atoi(e) != 0;
        if (const char* e = std::getenv("FMVS_SGM_AGG16"))
            ctx->agg16 = std::atoi(e) != 0;
        if (const char* e = std::getenv("FMVS_SGM_AGG16_MIN"))
            ctx->agg16_min = std::strtoull(e, nullptr, 10);
        if (const char* e = std::getenv("FMVS_SWEEP_STATS"))
            ctx->sweep_stats = std::atoi(e);  // 1: every level; 2 + l: level l only
        ctx->use();
        FMVS_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        {
            // keep stream-ordered temporaries (Tmp) in the pool across calls
            cudaMemPool_t pool;
            FMVS_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
            uint64_t keep = ~uint64_t(0);
            FMVS_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        }
        FMVS_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->staged, cudaEventDisableTiming));
        FMVS_CUDA_CHECK(cudaEventRecord(ctx->staged, ctx->stream));
        if (ctx->sweep_stats)
            FMVS_CUDA_CHECK(cudaMemset(ctx->buf("sweep_stats").as<unsigned long long>(8), 0, 64));
        *out = ctx.release();
    });
}

int32_t fmvs_current_device(void) {
    int d = -1;
    return cudaGetDevice(&d) == cudaSuccess ? d : -1;
}

void fmvs_ctx_destroy(fmvs_ctx* ctx) {
    if (!ctx)
        return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->bufs.clear();
    for (auto& sp : ctx->spans) {
        cudaEventDestroy(sp.a);
        cudaEventDestroy(sp.b);
    }
    for (cudaEvent_t e : ctx->event_pool)
        cudaEventDestroy(e);
    cudaEventDestroy(ctx->staged);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int fmvs_ctx_synchronize(fmvs_ctx* ctx) {
    return guarded([&] {
        ctx->use();
        FMVS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        finish_stats(ctx);
        ctx->collect();
    });
}

void fmvs_ctx_set_timing(fmvs_ctx* ctx, int32_t enable) { ctx->timing = enable != 0; }

// Diagnostics of the certified census sweep (FMVS_SWEEP_STATS=1): counts of
// (hypothesis, view) evaluations, evaluations with >= 1 undecided bit, undecided
// bits, exact-path views, tile-plane iterations run, tile-plane iterations
// skipped, exact samples taken, 0. Reads and clears the counters.
int fmvs_ctx_sweep_stats(fmvs_ctx* ctx, uint64_t out[8]) {
    return guarded([&] {
        ctx->use();
        for (int i = 0; i < 8; ++i)
            out[i] = 0;
        if (!ctx->sweep_stats)
            return;
        auto* d = ctx->buf("sweep_stats").as<unsigned long long>(8);
        FMVS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        FMVS_CUDA_CHECK(cudaMemcpy(out, d, 64, cudaMemcpyDeviceToHost));
        FMVS_CUDA_CHECK(cudaMemset(d, 0, 64));
    });
}

int fmvs_ctx_set_capture(fmvs_ctx* ctx, int32_t level) {
    ctx->cap = fmvs_ctx::Capture{};
    ctx->cap.level = level;
    return FMVS_OK;
}

int fmvs_ctx_capture_sizes(fmvs_ctx* ctx, int32_t* w, int32_t* h, uint64_t* entries) {
    return guarded([&] {
        if (ctx->cap.w == 0)
            fmvs::fail_input("capture: nothing captured");
        *w = ctx->cap.w;
        *h = ctx->cap.h;
        *entries = ctx->cap.costs.size();
    });
}

int fmvs_ctx_capture_copy(fmvs_ctx* ctx, int32_t* first, int32_t* count, uint64_t* offset,
                          uint16_t* costs, uint32_t* agg, int32_t* winners, float* depth_raw) {
    return guarded([&] {
        const auto& c = ctx->cap;
        if (c.w == 0)
            fmvs::fail_input("capture: nothing captured");
        for (int y = 0; y < c.h; ++y)
            for (int x = 0; x < c.w; ++x) {
                const size_t p = static_cast<size_t>(y) * c.w + x;
                first[p] = static_cast<int32_t>(c.meta[p].fc & 0xffffu);
                count[p] = static_cast<int32_t>(c.meta[p].fc >> 16);
                offset[p] = c.row_base[y] + c.meta[p].rel;
            }
        std::copy(c.costs.begin(), c.costs.end(), costs);
        std::copy(c.agg.begin(), c.agg.end(), agg);
        std::copy(c.winners.begin(), c.winners.end(), winners);
        std::copy(c.depth_raw.begin(), c.depth_raw.end(), depth_raw);
    });
}

int32_t fmvs_ctx_stage_count(fmvs_ctx* ctx) { return static_cast<int32_t>(ctx->stage_names.size()); }

const char* fmvs_ctx_stage_name(fmvs_ctx* ctx, int32_t i) {
    return i >= 0 && i < static_cast<int32_t>(ctx->stage_names.size()) ? ctx->stage_names[i].c_str() : "";
}

int fmvs_ctx_stage_time(fmvs_ctx* ctx, int32_t i, double* ms, int64_t* calls) {
    if (i < 0 || i >= static_cast<int32_t>(ctx->stage_names.size()))
        return FMVS_ERR_INVALID_INPUT;
    *ms = ctx->stage_ms[i];
    *calls = ctx->stage_calls[i];
    return FMVS_OK;
}

void fmvs_ctx_stage_reset(fmvs_ctx* ctx) {
    std::fill(ctx->stage_ms.begin(), ctx->stage_ms.end(), 0.0);
    std::fill(ctx->stage_calls.begin(), ctx->stage_calls.end(), 0);
}

int32_t fmvs_ctx_level_stats(fmvs_ctx* ctx, fmvs_level_stats* out, int32_t capacity) {
    const int32_t n = std::min<int32_t>(capacity, static_cast<int32_t>(ctx->stats.size()));
    for (int32_t i = 0; i < n; ++i)
        out[i] = ctx->stats[i];
    return n;
}

int64_t fmvs_ctx_last_launch_count(fmvs_ctx* ctx) { return ctx->launches; }

void* fmvs_ctx_stream(fmvs_ctx* ctx) { return ctx->stream; }

void* fmvs_host_alloc(uint64_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess)
        return nullptr;
    return p;
}

void fmvs_host_free(void* p) {
    if (p)
        cudaFreeHost(p);
}

int fmvs_estimate_bundle(fmvs_ctx* ctx, const fmvs_view* views, int32_t n, const fmvs_config* cfg,
                         float* depth, float* normals_xyz, float* confidence) {
    return guarded([&] {
        ctx->use();
        if (!cfg)
            fmvs::fail_config("estimate: null config");
        fmvs::validate_config(*cfg);
        if (n < 3 || n % 2 == 0)
            fmvs::fail_input("estimate: bundle must hold an odd number (>= 3) of views");
        for (int i = 0; i < n; ++i)
            fmvs::validate_view(views[i]);
        std::vector<const uint8_t*> d_images;
        copy_views_to_device(ctx, views, n, &d_images);
        const fmvs_intrinsics& k0 = views[n / 2].intrinsics;
        const size_t px = static_cast<size_t>(k0.width) * k0.height;
        float* d_out = ctx->buf("host_out").as<float>(5 * px);
        run_bundle(ctx, views, n, *cfg, d_images.data(), d_out, d_out + px, d_out + 4 * px);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(depth, d_out, px * 4, cudaMemcpyDeviceToHost, ctx->stream));
        FMVS_CUDA_CHECK(cudaMemcpyAsync(normals_xyz, d_out + px, 3 * px * 4, cudaMemcpyDeviceToHost, ctx->stream));
        FMVS_CUDA_CHECK(cudaMemcpyAsync(confidence, d_out + 4 * px, px * 4, cudaMemcpyDeviceToHost, ctx->stream));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        finish_stats(ctx);
        ctx->collect();
    });
}

int fmvs_estimate_bundle_device(fmvs_ctx* ctx, const fmvs_view* views, int32_t n,
                                const fmvs_config* cfg, float* d_depth, float* d_normals_xyz,
                                float* d_confidence) {
    return guarded([&] {
        ctx->use();
        if (!cfg)
            fmvs::fail_config("estimate: null config");
        std::vector<const uint8_t*> d_images(std::max(n, 0));
        for (int i = 0; i < n; ++i)
            d_images[i] = views[i].image;
        run_bundle(ctx, views, n, *cfg, d_images.data(), d_depth, d_normals_xyz, d_confidence);
    });
}

// -------------------------------------------------------- host geometry --

int fmvs_plane_homography(const double normal[3], double distance, const fmvs_intrinsics* ri,
                          const fmvs_pose* rp, const fmvs_intrinsics* oi, const fmvs_pose* op,
                          double out_h[9]) {
    return guarded([&] {
        const fmvs::M3 H = fmvs::plane_homography(v3(normal), distance, fmvs::camera_of(*ri, *rp),
                                                  fmvs::camera_of(*oi, *op));
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                out_h[3 * r + c] = H.a[r][c];
    });
}

int fmvs_bounding_distances(double d_min, double d_max, const double normal[3],
                            const fmvs_intrinsics* ri, double* lo, double* hi) {
    return guarded([&] { fmvs::bounding_distances(d_min, d_max, v3(normal), *ri, lo, hi); });
}

int fmvs_plane_distances(const fmvs_intrinsics* ri, const fmvs_pose* rp, const fmvs_intrinsics* oi,
                         const fmvs_pose* op, double delta_min, double delta_max,
                         const double normal[3], int32_t max_planes, double* out, int32_t capacity,
                         int32_t* count) {
    int rc = guarded([&] {
        const std::vector<double> d =
            fmvs::plane_distances(fmvs::camera_of(*ri, *rp), fmvs::camera_of(*oi, *op), delta_min,
                                  delta_max, v3(normal), max_planes);
        *count = static_cast<int32_t>(d.size());
        for (int i = 0; i < static_cast<int>(d.size()) && i < capacity; ++i)
            out[i] = d[i];
    });
    if (rc == FMVS_OK && *count > capacity) {
        g_last_error = "plane distances: output capacity too small";
        return FMVS_ERR_CAPACITY;
    }
    return rc;
}

double fmvs_depth_from_plane(double x, double y, const double normal[3], double distance,
                             const fmvs_intrinsics* intr) {
    return fmvs::depth_from_plane(x, y, v3(normal), distance, *intr);
}

double fmvs_adaptive_phi2(double phi1, double alpha, double beta, double di) {
    return fmvs::adaptive_phi2(phi1, alpha, beta, di);
}

int fmvs_parabola_refine(double a, double b, double c, double ca, double cb, double cc,
                         double* out) {
    return guarded([&] { *out = fmvs::parabola_refine(a, b, c, ca, cb, cc); });
}

// --------------------------------------------------------- device stages --

int fmvs_build_pyramids(fmvs_ctx* ctx, const fmvs_view* views, int32_t n, int32_t levels,
                        uint8_t* out_images, uint64_t capacity, fmvs_intrinsics* out_intr) {
    return guarded([&] {
        ctx->use();
        if (levels < 1)
            fmvs::fail_config("pyramids: need at least one level");
        for (int i = 0; i < n; ++i)
            fmvs::validate_view(views[i]);
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        std::vector<fmvs_intrinsics> intr(static_cast<size_t>(levels) * n);
        std::vector<uint8_t*> d(static_cast<size_t>(levels) * n);
        uint64_t need = 0;
        for (int l = 0; l < levels; ++l)
            for (int k2 = 0; k2 < n; ++k2) {
                intr[l * n + k2] = l == 0 ? views[k2].intrinsics : fmvs::halved(intr[(l - 1) * n + k2]);
                const size_t px = static_cast<size_t>(intr[l * n + k2].width) * intr[l * n + k2].height;
                need += px;
                d[l * n + k2] = l == 0 ? t.upload(views[k2].image, px, s) : t.alloc<uint8_t>(px);
            }
        if (need > capacity)
            throw fmvs::Error(FMVS_ERR_CAPACITY, "pyramids: output capacity too small");
        double k3[3];
        fmvs::blur3_kernel(k3);
        for (int l = 1; l < levels; ++l)
            for (int k2 = 0; k2 < n; ++k2) {
                const auto& a = intr[(l - 1) * n + k2];
                const auto& b = intr[l * n + k2];
                k::blur_halve(d[(l - 1) * n + k2], a.width, a.height, d[l * n + k2], b.width,
                              b.height, k3, s);
            }
        uint64_t pos = 0;
        for (int l = 0; l < levels; ++l)
            for (int k2 = 0; k2 < n; ++k2) {
                const size_t px = static_cast<size_t>(intr[l * n + k2].width) * intr[l * n + k2].height;
                FMVS_CUDA_CHECK(cudaMemcpyAsync(out_images + pos, d[l * n + k2], px, cudaMemcpyDeviceToHost, s));
                pos += px;
                out_intr[l * n + k2] = intr[l * n + k2];
            }
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int fmvs_refine_range(fmvs_ctx* ctx, const float* prior, int32_t w, int32_t h, int32_t kind,
                      double value, double d_min, double d_max, const fmvs_plane_stack* coarser,
                      const fmvs_intrinsics* intr, float* lo, float* hi) {
    return guarded([&] {
        ctx->use();
        fmvs::validate_depth_bounds(d_min, d_max);
        if (kind == FMVS_RANGE_SPACING_MULTIPLE && (!coarser || !intr || coarser->count < 2))
            fmvs::fail_config("refine range: spacing policy needs the coarser plane stack");
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const size_t px = static_cast<size_t>(w) * h;
        k::RangeArgs ra{};
        fmvs_intrinsics k0 = intr ? *intr : fmvs_intrinsics{1, 1, 0, 0, w, h};
        k0.width = w;
        k0.height = h;
        ra.intr = intr_of(k0);
        ra.nx = coarser ? coarser->normal[0] : 0;
        ra.ny = coarser ? coarser->normal[1] : 0;
        ra.nz = coarser ? coarser->normal[2] : -1;
        const double one = 1.0;
        ra.planes = t.upload(&one, 1, s);
        ra.nplanes = 1;
        ra.mode = 1;
        ra.d_min = d_min;
        ra.d_max = d_max;
        ra.prior = t.upload(prior, px, s);
        ra.prior_w = w;
        ra.prior_h = h;
        ra.policy = kind;
        ra.policy_value = value;
        if (coarser) {
            ra.coarser = t.upload(coarser->distances, coarser->count, s);
            ra.ncoarser = coarser->count;
        }
        ra.lo_out = t.alloc<float>(px);
        ra.hi_out = t.alloc<float>(px);
        ra.meta = t.alloc<fmvs::dev::VolMeta>(px);
        ra.row_total = t.alloc<uint32_t>(h);
        k::range_rows(ra, s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(lo, ra.lo_out, px * 4, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaMemcpyAsync(hi, ra.hi_out, px * 4, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int fmvs_sweep_cost_volume(fmvs_ctx* ctx, const fmvs_view* views, int32_t n, int32_t ref_index,
                           const fmvs_plane_stack* planes, const float* lo, const float* hi,
                           const fmvs_cost_spec* cost, int32_t* first, int32_t* count,
                           uint64_t* offset, uint16_t* costs, uint64_t capacity, uint64_t* total,
                           int32_t* per_side) {
    int rc = guarded([&] {
        ctx->use();
        fmvs::validate_cost(*cost);  // matching.cpp:119-142
        if (ref_index < 0 || ref_index >= n)
            fmvs::fail_input("sweep: reference index out of range");
        if (ref_index < 1 || ref_index > n - 2)
            fmvs::fail_input("sweep: need at least one matching image on each side");
        for (int i = 0; i < n; ++i)
            fmvs::validate_view(views[i]);
        if (planes->count < 1)
            fmvs::fail_input("sweep: empty plane list");
        for (int i = 1; i < planes->count; ++i)
            if (!(planes->distances[i] < planes->distances[i - 1]))
                fmvs::fail_input("sweep: plane distances must be strictly decreasing");
        if (planes->count > 65535)
            fmvs::fail_config("b200: more than 65535 sweep planes in one level is unsupported");
        const fmvs::Camera cref = fmvs::camera_of(views[ref_index]);
        std::vector<fmvs::V3> centers;
        for (int k2 = 0; k2 < n; ++k2)
            centers.push_back(fmvs::mul(cref.rot, fmvs::sub(fmvs::camera_of(views[k2]).center, cref.center)));
        const fmvs::V3 normal = v3(planes->normal);
        fmvs::require_centers_in_front(normal, planes->distances[planes->count - 1], centers);
        *per_side = std::max(ref_index, n - 1 - ref_index);

        const int w = views[ref_index].intrinsics.width, h = views[ref_index].intrinsics.height;
        const size_t px = static_cast<size_t>(w) * h;
        const int np = planes->count;
        std::vector<double> homs(static_cast<size_t>(n - 1) * np * 9);
        std::vector<const uint32_t*> qptr;
        std::vector<int2> sizes;
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        int m = 0;
        for (int k2 = 0; k2 < n; ++k2) {
            if (k2 == ref_index)
                continue;
            const fmvs::Camera ck = fmvs::camera_of(views[k2]);
            for (int i = 0; i < np; ++i) {
                const fmvs::M3 H = fmvs::plane_homography(normal, planes->distances[i], cref, ck);
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c)
                        homs[(static_cast<size_t>(m) * np + i) * 9 + 3 * r + c] = H.a[r][c];
            }
            const int vw = views[k2].intrinsics.width, vh = views[k2].intrinsics.height;
            const size_t vpx = static_cast<size_t>(vw) * vh;
            uint8_t* di = t.upload(views[k2].image, vpx, s);
            uint32_t* dq = t.alloc<uint32_t>(vpx);
            k::pack_quads(di, vw, vh, dq, s);
            qptr.push_back(dq);
            sizes.push_back(make_int2(vw, vh));
            ++m;
        }
        k::RangeArgs ra{};
        ra.intr = intr_of(views[ref_index].intrinsics);
        ra.nx = normal.x;
        ra.ny = normal.y;
        ra.nz = normal.z;
        ra.planes = t.upload(planes->distances, np, s);
        ra.nplanes = np;
        ra.mode = 2;
        ra.lo_in = t.upload(lo, px, s);
        ra.hi_in = t.upload(hi, px, s);
        ra.meta = t.alloc<fmvs::dev::VolMeta>(px);
        ra.row_total = t.alloc<uint32_t>(h);
        k::range_rows(ra, s);
        uint64_t* rb = t.alloc<uint64_t>(h + 1);
        k::scan_rows(ra.row_total, h, rb, s);
        std::vector<uint64_t> h_rb(h + 1);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(h_rb.data(), rb, (h + 1) * 8, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
        *total = h_rb[h];
        const uint64_t ne = h_rb[h];
        k::SweepArgs sa{};
        sa.w = w;
        sa.h = h;
        sa.ref_img = t.upload(views[ref_index].image, px, s);
        sa.nmatch = n - 1;
        sa.quads = t.upload(qptr.data(), qptr.size(), s);
        sa.sizes = t.upload(sizes.data(), sizes.size(), s);
        sa.homs = t.upload(homs.data(), homs.size(), s);
        sa.nplanes = np;
        sa.nleft = ref_index;
        sa.meta = ra.meta;
        sa.row_base = rb;
        sa.costs = t.alloc<uint16_t>(ne);
        sa.kind = cost->kind;
        sa.ww = cost->window_w;
        sa.wh = cost->window_h;
        const std::vector<uint16_t> clut = fmvs::census_cost_table(cost->window_w * cost->window_h - 1);
        sa.census_lut = t.upload(clut.data(), clut.size(), s);
        sa.plane_slicing = 1;
        if (const char* e = std::getenv("FMVS_SWEEP_NARROW"))
            sa.narrow_max = std::atoi(e);
        sa.small_lists = std::getenv("FMVS_NCC_SMALL_LISTS") != nullptr;
        k::sweep(sa, s);
        std::vector<fmvs::dev::VolMeta> meta(px);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(meta.data(), ra.meta, px * 8, cudaMemcpyDeviceToHost, s));
        if (ne <= capacity && ne > 0)
            FMVS_CUDA_CHECK(cudaMemcpyAsync(costs, sa.costs, ne * 2, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                const size_t p = static_cast<size_t>(y) * w + x;
                first[p] = static_cast<int32_t>(meta[p].fc & 0xFFFFu);
                count[p] = static_cast<int32_t>(meta[p].fc >> 16);
                offset[p] = h_rb[y] + meta[p].rel;
            }
    });
    if (rc == FMVS_OK && *total > capacity) {
        g_last_error = "sweep: cost capacity too small";
        return FMVS_ERR_CAPACITY;
    }
    return rc;
}

int fmvs_compute_normal_offsets(fmvs_ctx* ctx, const float* prior_normals_xyz,
                                const float* prior_depth, int32_t w, int32_t h,
                                const fmvs_plane_stack* planes, const fmvs_intrinsics* intr,
                                int16_t* out) {
    return guarded([&] {
        ctx->use();
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const size_t px = static_cast<size_t>(w) * h;
        k::OffsetArgs oa{};
        fmvs_intrinsics k0 = *intr;
        oa.intr = intr_of(k0);
        oa.w = w;
        oa.h = h;
        oa.prior_depth = t.upload(prior_depth, px, s);
        oa.prior_normals = t.upload(prior_normals_xyz, 3 * px, s);
        oa.prior_w = w;
        oa.prior_h = h;
        oa.nx = planes->normal[0];
        oa.ny = planes->normal[1];
        oa.nz = planes->normal[2];
        oa.planes = t.upload(planes->distances, planes->count, s);
        oa.nplanes = planes->count;
        oa.out = t.alloc<int16_t>(4 * px);
        k::normal_offsets(oa, s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(out, oa.out, px * 8, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

}  // extern "C"

namespace {

// aggregate (all cfg->paths directions) or aggregate_single_path (one step
// (dir_x, dir_y), any integers; sgm.cpp:301-331) on a host-given volume.
int aggregate_impl(fmvs_ctx* ctx, int32_t w, int32_t h, const fmvs_plane_stack* planes,
                   const int32_t* first, const int32_t* count, const uint64_t* offset,
                   const uint16_t* costs, uint64_t total, const uint8_t* image,
                   const fmvs_sgm_config* cfg, const fmvs_intrinsics* intr,
                   const float* prior_normals_xyz, const float* prior_depth, bool all_paths,
                   int32_t dir_x, int32_t dir_y, uint32_t* out_values) {
    return guarded([&] {
        ctx->use();
        fmvs::validate_sgm(*cfg);  // check_aggregate_inputs, sgm.cpp:241-248
        if (cfg->variant == FMVS_SGM_SURFACE_NORMAL && (!prior_normals_xyz || !prior_depth))
            fmvs::fail_config("sgm: surface-normal variant requires a prior normal and depth map");
        static const int kDirs[8][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1},
                                        {1, 1}, {-1, -1}, {1, -1}, {-1, 1}};
        k::SgmArgs ga{};
        if (all_paths) {
            ga.ndirs = cfg->paths == 8 ? 8 : 4;
            for (int d = 0; d < 8; ++d) {
                ga.dirs[d][0] = kDirs[d][0];
                ga.dirs[d][1] = kDirs[d][1];
            }
        } else {
            ga.ndirs = 1;
            ga.dirs[0][0] = dir_x;
            ga.dirs[0][1] = dir_y;
        }
        std::vector<fmvs::dev::VolMeta> meta;
        std::vector<uint64_t> rb, src;
        uint64_t n_entries = 0;
        host_layout(w, h, first, count, offset, total, &meta, &rb, &src, &n_entries);
        std::vector<uint16_t> gathered;
        if (!src.empty()) {
            gathered = gather(costs, src);
            costs = gathered.data();
        }
        const uint64_t stored = total;  // the caller's value array (zeros outside pixel ranges)
        total = n_entries;
        if (!all_paths && cfg->variant == FMVS_SGM_SURFACE_NORMAL) {
            // The SN shift exists only along the canonical directions and
            // their opposites; the reference throws when a line takes a step
            // between two non-empty pixels along another one (sgm.cpp:72-80,
            // 129-130).
            const int ax = std::abs(dir_x), ay = std::abs(dir_y);
            const bool canonical = ax <= 1 && ay <= 1 && (ax | ay) != 0;
            if (!canonical)
                for (int y = 0; y < h; ++y)
                    for (int x = 0; x < w; ++x) {
                        const int px2 = x - dir_x, py2 = y - dir_y;
                        if (count[static_cast<size_t>(y) * w + x] > 0 && px2 >= 0 && py2 >= 0 && px2 < w &&
                            py2 < h && count[static_cast<size_t>(py2) * w + px2] > 0)
                            fmvs::fail_config("sgm: unsupported path direction");
                    }
        }
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const size_t px = static_cast<size_t>(w) * h;
        int pmax = 1;
        for (size_t p = 0; p < px; ++p)
            pmax = std::max(pmax, static_cast<int>(count[p]));
        ga.w = w;
        ga.h = h;
        ga.meta = t.upload(meta.data(), px, s);
        ga.row_base = t.upload(rb.data(), rb.size(), s);
        ga.costs = t.upload(costs, total, s);
        ga.agg = t.alloc<uint32_t>(total + k::kAggSlack);
        ga.cost_max = total > 0 ? static_cast<int>(*std::max_element(costs, costs + total)) : -1;
        FMVS_CUDA_CHECK(cudaMemsetAsync(ga.agg, 0, std::max<uint64_t>(total, 1) * 4, s));
        ga.image = t.upload(image, px, s);
        ga.variant = cfg->variant;
        ga.phi1 = std::llround(cfg->phi1 * cfg->penalty_scale);
        const std::vector<long long> lut = fmvs::phi2_table(*cfg);
        ga.phi2_lut = t.upload(lut.data(), lut.size(), s);
        ga.phi2_max = *std::max_element(lut.begin(), lut.end());
        ga.intr = intr_of(*intr);
        ga.nx = planes->normal[0];
        ga.ny = planes->normal[1];
        ga.nz = planes->normal[2];
        ga.planes = t.upload(planes->distances, planes->count, s);
        ga.nplanes = planes->count;
        if (cfg->variant == FMVS_SGM_SURFACE_NORMAL) {
            k::OffsetArgs oa{};
            oa.intr = ga.intr;
            oa.w = w;
            oa.h = h;
            oa.prior_depth = t.upload(prior_depth, px, s);
            oa.prior_normals = t.upload(prior_normals_xyz, 3 * px, s);
            oa.prior_w = w;
            oa.prior_h = h;
            oa.nx = ga.nx;
            oa.ny = ga.ny;
            oa.nz = ga.nz;
            oa.planes = ga.planes;
            oa.nplanes = ga.nplanes;
            oa.out = t.alloc<int16_t>(4 * px);
            k::normal_offsets(oa, s);
            ga.offsets = oa.out;
        }
        ga.pmax = pmax;
        sgm_blocking(&ga.group, &ga.kper, pmax);
        ga.group_caps = 32;
        const int limit = (200 * 1024) / (4 * 2 * 4);
        if (pmax > limit || ga.group > 0) {
            const size_t lines = static_cast<size_t>(k::sgm_lines(w, h, ga.dirs, ga.ndirs));
            ga.scratch = t.alloc<uint32_t>(lines * 2 * (pmax + k::kSgmLinePad));
        }
        ga.line_scratch = t.alloc<uint32_t>(k::sgm_line_scratch_words(w, h));
        ga.entries_bound = total;
        if (total > 0)
            k::sgm(ga, s);
        std::vector<uint32_t> compact_out;
        const bool remap = !src.empty() || total != stored;
        uint32_t* dst = out_values;
        if (remap) {
            compact_out.resize(total);
            dst = compact_out.data();
        }
        if (total > 0)
            FMVS_CUDA_CHECK(cudaMemcpyAsync(dst, ga.agg, total * 4, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
        if (remap) {  // make_accumulator zeroes the whole array (sgm.cpp:198-208)
            std::fill(out_values, out_values + stored, 0u);
            for (size_t i = 0; i < compact_out.size(); ++i)
                out_values[src.empty() ? i : src[i]] = compact_out[i];
        }
    });
}

}  // namespace

extern "C" {

int fmvs_aggregate(fmvs_ctx* ctx, int32_t w, int32_t h, const fmvs_plane_stack* planes,
                   const int32_t* first, const int32_t* count, const uint64_t* offset,
                   const uint16_t* costs, uint64_t total, const uint8_t* image,
                   const fmvs_sgm_config* cfg, const fmvs_intrinsics* intr,
                   const float* prior_normals_xyz, const float* prior_depth, int32_t dir_x,
                   int32_t dir_y, uint32_t* out_values) {
    return aggregate_impl(ctx, w, h, planes, first, count, offset, costs, total, image, cfg, intr,
                          prior_normals_xyz, prior_depth, dir_x == 0 && dir_y == 0, dir_x, dir_y,
                          out_values);
}

int fmvs_aggregate_single_path(fmvs_ctx* ctx, int32_t w, int32_t h, const fmvs_plane_stack* planes,
                               const int32_t* first, const int32_t* count, const uint64_t* offset,
                               const uint16_t* costs, uint64_t total, const uint8_t* image,
                               const fmvs_sgm_config* cfg, const fmvs_intrinsics* intr,
                               const float* prior_normals_xyz, const float* prior_depth,
                               int32_t dir_x, int32_t dir_y, uint32_t* out_values) {
    return aggregate_impl(ctx, w, h, planes, first, count, offset, costs, total, image, cfg, intr,
                          prior_normals_xyz, prior_depth, false, dir_x, dir_y, out_values);
}

int fmvs_wta(fmvs_ctx* ctx, int32_t w, int32_t h, const int32_t* first, const int32_t* count,
             const uint64_t* offset, const uint32_t* values, uint64_t total, int32_t* winners) {
    return guarded([&] {
        ctx->use();
        std::vector<fmvs::dev::VolMeta> meta;
        std::vector<uint64_t> rb, src;
        uint64_t n_entries = 0;
        host_layout(w, h, first, count, offset, total, &meta, &rb, &src, &n_entries);
        std::vector<uint32_t> gathered;
        if (!src.empty()) {
            gathered = gather(values, src);
            values = gathered.data();
        }
        total = n_entries;
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const size_t px = static_cast<size_t>(w) * h;
        k::WtaArgs wa{};
        wa.w = w;
        wa.h = h;
        wa.meta = t.upload(meta.data(), px, s);
        wa.row_base = t.upload(rb.data(), rb.size(), s);
        wa.agg = t.upload(values, total, s);
        wa.winners = t.alloc<int32_t>(px);
        if (px > 0)
            k::wta_depth(wa, s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(winners, wa.winners, px * 4, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int fmvs_median_filter_5x5(fmvs_ctx* ctx, const float* depth, int32_t w, int32_t h, float* out) {
    return guarded([&] {
        ctx->use();
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const size_t px = static_cast<size_t>(w) * h;
        const float* din = t.upload(depth, px, s);
        float* dout = t.alloc<float>(px);
        if (px > 0)
            k::median5(din, w, h, dout, s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(out, dout, px * 4, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int fmvs_normals_from_depth(fmvs_ctx* ctx, const float* depth, int32_t w, int32_t h,
                            const fmvs_intrinsics* intr, float* out_xyz) {
    return guarded([&] {
        ctx->use();
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const size_t px = static_cast<size_t>(w) * h;
        const float* din = t.upload(depth, px, s);
        float* dout = t.alloc<float>(3 * px);
        if (px > 0)
            k::normals_raw(din, w, h, intr_of(*intr), dout, s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(out_xyz, dout, 3 * px * 4, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int fmvs_smooth_normals(fmvs_ctx* ctx, const float* raw_xyz, const uint8_t* image, int32_t w,
                        int32_t h, int32_t radius, float* out_xyz) {
    return guarded([&] {
        ctx->use();
        if (radius < 1)  // surface.cpp:42-45
            fmvs::fail_config("smooth normals: radius must be at least 1");
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const size_t px = static_cast<size_t>(w) * h;
        const std::vector<double> wt = fmvs::smoothing_table(radius);
        const float* din = t.upload(raw_xyz, 3 * px, s);
        const uint8_t* dimg = t.upload(image, px, s);
        const double* dwt = t.upload(wt.data(), wt.size(), s);
        float* dout = t.alloc<float>(3 * px);
        if (px > 0)
            k::smooth_conf(din, dimg, w, h, radius, dwt, dout, nullptr, 0, 0, 0, 0, 0, s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(out_xyz, dout, 3 * px * 4, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int fmvs_confidence_map(fmvs_ctx* ctx, const float* normals_xyz, int32_t w, int32_t h,
                        const double sweep_normal[3], double rho_degrees, float* out) {
    return guarded([&] {
        ctx->use();
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const size_t px = static_cast<size_t>(w) * h;
        const double cos_rho = std::cos(rho_degrees * M_PI / 180.0);  // surface.cpp:85-87
        const double pdv = (sweep_normal[0] * 0.0 + sweep_normal[1] * 0.0) + sweep_normal[2] * -1.0;
        const float* din = t.upload(normals_xyz, 3 * px, s);
        float* dout = t.alloc<float>(px);
        if (px > 0)
            k::confidence(din, w, h, cos_rho, pdv, sweep_normal[0], sweep_normal[1], sweep_normal[2],
                          dout, s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(out, dout, px * 4, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int fmvs_upscale_nearest(fmvs_ctx* ctx, const float* in, int32_t iw, int32_t ih, int32_t ch,
                         int32_t ow, int32_t oh, float* out) {
    return guarded([&] {
        ctx->use();
        if (ow == iw && oh == ih) {  // identity (pipeline.cpp:93-94)
            std::memcpy(out, in, sizeof(float) * ch * static_cast<size_t>(iw) * ih);
            return;
        }
        if ((iw + 1) / 2 > ow || (ih + 1) / 2 > oh)
            fmvs::fail_input("upscale: target smaller than the source level");
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const float* din = t.upload(in, static_cast<size_t>(ch) * iw * ih, s);
        float* dout = t.alloc<float>(static_cast<size_t>(ch) * ow * oh);
        k::upscale(din, iw, ih, ch, dout, ow, oh, s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(out, dout, sizeof(float) * ch * static_cast<size_t>(ow) * oh,
                                        cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int fmvs_render_scene(fmvs_ctx* ctx, const fmvs_scene_plane* planes, int32_t n_planes,
                      const fmvs_pose* poses, int32_t n_poses, const fmvs_intrinsics* intrinsics,
                      int32_t texture, double texture_scale, uint64_t seed, uint8_t* images,
                      float* gt_depth, float* gt_normals_xyz) {
    return guarded([&] {
        ctx->use();
        // render_scene (render.cpp:52-141): validation in the reference's order
        const fmvs_intrinsics k0 = *intrinsics;
        fmvs::validate_intrinsics(k0);
        if (n_planes < 1 || n_poses < 1)
            fmvs::fail_input("render: scene needs at least one plane and one pose");
        if (!(texture_scale > 0.0))
            fmvs::fail_input("render: texture scale must be positive");
        if (texture != FMVS_TEXTURE_CHECKERBOARD && texture != FMVS_TEXTURE_VALUE_NOISE)
            fmvs::fail_input("render: unknown texture kind");
        // PlaneFrame (render.cpp:64-72): Eigen normalized() leaves a zero vector as is
        auto normalized = [](fmvs::V3 v) {
            const double n2 = fmvs::dot(v, v);
            return n2 > 0.0 ? fmvs::divs(v, std::sqrt(n2)) : v;
        };
        std::vector<k::RenderPlane> frames(n_planes);
        for (int i = 0; i < n_planes; ++i) {
            const fmvs_scene_plane& sp = planes[i];
            const fmvs::V3 fn = normalized(fmvs::V3{sp.normal[0], sp.normal[1], sp.normal[2]});
            const fmvs::V3 u0{sp.u_axis[0], sp.u_axis[1], sp.u_axis[2]};
            const fmvs::V3 fu = normalized(fmvs::sub(u0, fmvs::scale(fmvs::dot(u0, fn), fn)));
            const fmvs::V3 fv = fmvs::cross(fn, fu);
            k::RenderPlane& f = frames[i];
            for (int c = 0; c < 3; ++c)
                f.pt[c] = sp.point[c];
            f.n[0] = fn.x, f.n[1] = fn.y, f.n[2] = fn.z;
            f.u[0] = fu.x, f.u[1] = fu.y, f.u[2] = fu.z;
            f.v[0] = fv.x, f.v[1] = fv.y, f.v[2] = fv.z;
            f.ext_u = sp.extent_u;
            f.ext_v = sp.extent_v;
        }
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const size_t px = static_cast<size_t>(k0.width) * k0.height;
        k::RenderPlane* dplanes = t.upload(frames.data(), frames.size(), s);
        uint8_t* dimg = t.alloc<uint8_t>(px * n_poses);
        float* dd = gt_depth ? t.alloc<float>(px * n_poses) : nullptr;
        float* dn = gt_normals_xyz ? t.alloc<float>(3 * px * n_poses) : nullptr;
        for (int v = 0; v < n_poses; ++v) {
            fmvs::validate_pose(fmvs::camera_of(k0, poses[v]).rot);  // pose.validate() per view
            k::RenderArgs ra{};
            ra.w = k0.width;
            ra.h = k0.height;
            ra.intr = intr_of(k0);
            std::memcpy(ra.rot, poses[v].rotation, sizeof(ra.rot));
            std::memcpy(ra.center, poses[v].center, sizeof(ra.center));
            ra.planes = dplanes;
            ra.nplanes = n_planes;
            ra.texture = texture;
            ra.texture_scale = texture_scale;
            ra.seed = seed;
            ra.image = dimg + v * px;
            ra.gt_depth = dd ? dd + v * px : nullptr;
            ra.gt_normals = dn ? dn + 3 * v * px : nullptr;
            k::render_view(ra, s);
        }
        FMVS_CUDA_CHECK(cudaMemcpyAsync(images, dimg, px * n_poses, cudaMemcpyDeviceToHost, s));
        if (dd)
            FMVS_CUDA_CHECK(cudaMemcpyAsync(gt_depth, dd, 4 * px * n_poses, cudaMemcpyDeviceToHost, s));
        if (dn)
            FMVS_CUDA_CHECK(cudaMemcpyAsync(gt_normals_xyz, dn, 12 * px * n_poses, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int fmvs_render_plane_scene(fmvs_ctx* ctx, int32_t kind, int32_t w, int32_t h, double focal,
                            double depth, double tilt_deg, int32_t n_views, double step,
                            uint64_t seed, double texture_scale, uint8_t* images, float* gt_depth,
                            float* gt_normals_xyz, fmvs_intrinsics* intr, fmvs_pose* poses) {
    // base_scene / fronto_scene / slanted_scene (render.cpp:143-183)
    const fmvs_intrinsics k0{focal, focal, (w - 1) / 2.0, (h - 1) / 2.0, w, h};
    const double inf = std::numeric_limits<double>::infinity();
    fmvs_scene_plane plane{{0, 0, depth}, {0, 0, -1}, {1, 0, 0}, inf, inf};
    if (kind == 1) {
        const double rad = tilt_deg * M_PI / 180.0;
        plane.normal[1] = -std::sin(rad);
        plane.normal[2] = -std::cos(rad);
        plane.normal[0] = 0.0;
    }
    std::vector<fmvs_pose> ps(n_views > 0 ? n_views : 0);
    for (int v = 0; v < n_views; ++v) {
        fmvs_pose pose{};
        pose.rotation[0] = pose.rotation[4] = pose.rotation[8] = 1.0;
        pose.center[0] = (v - (n_views - 1) / 2.0) * step;  // lateral_trajectory
        ps[v] = pose;
        if (intr)
            intr[v] = k0;
        if (poses)
            poses[v] = pose;
    }
    return fmvs_render_scene(ctx, &plane, 1, ps.data(), n_views, &k0, FMVS_TEXTURE_VALUE_NOISE,
                             texture_scale, seed, images, gt_depth, gt_normals_xyz);
}

}  // extern "C"

// ------------------------------------------------ post-filters (§8f) --
namespace {

// DoG texture mask of a device image (postfilter.cpp:67-79) into d_mask.
void dog_mask_device(fmvs_ctx* ctx, const uint8_t* d_img, int w, int h, uint8_t* d_mask) {
    cudaStream_t s = ctx->stream;
    const size_t px = static_cast<size_t>(w) * h;
    const std::vector<double> kw = fmvs::blur_kernel(3, 1.4);
    k::BlurKernel bk{};
    bk.radius = 3;
    for (size_t i = 0; i < kw.size(); ++i)
        bk.w[i] = kw[i];
    float* tmp = ctx->buf("dog_tmp").as<float>(px);
    int* labels = ctx->buf("dog_labels").as<int>(px);
    int* sizes = ctx->buf("dog_sizes").as<int>(px);
    uint8_t* act = ctx->buf("dog_act").as<uint8_t>(px);
    k::gaussian_blur_dog(d_img, w, h, bk, tmp, act, s);
    k::remove_speckles(act, w, h, 1, 7, labels, sizes, s);
    k::dilate3(act, w, h, d_mask, s);
    k::remove_speckles(d_mask, w, h, 0, 21, labels, sizes, s);
}

void check_geom_window(int n, int ref_index, const fmvs_geom_filter_config& c) {
    if (c.eta_h < 1 || n < c.eta_h + 1)  // postfilter.cpp:97-100
        fmvs::fail_config("geometric filter: window smaller than eta_h + 1 views");
    if (ref_index < 0 || ref_index >= n)
        fmvs::fail_input("geometric filter: reference index out of range");
}

k::GeomView geom_view(const float* d_depth, int w, int h, const fmvs_intrinsics& k0,
                      const fmvs_pose& pose) {
    k::GeomView g{};
    g.depth = d_depth;
    g.w = w;
    g.h = h;
    g.k = intr_of(k0);
    for (int i = 0; i < 9; ++i)
        g.R[i] = pose.rotation[i];
    for (int i = 0; i < 3; ++i)
        g.C[i] = pose.center[i];
    return g;
}

}  // namespace

extern "C" {

int fmvs_dog_mask(fmvs_ctx* ctx, const uint8_t* image, int32_t w, int32_t h, uint8_t* out) {
    return guarded([&] {
        ctx->use();
        if (w <= 0 || h <= 0)
            return;
        const size_t px = static_cast<size_t>(w) * h;
        Tmp t(ctx->stream);
        const uint8_t* d_img = t.upload(image, px, ctx->stream);
        uint8_t* d_mask = t.alloc<uint8_t>(px);
        dog_mask_device(ctx, d_img, w, h, d_mask);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(out, d_mask, px, cudaMemcpyDeviceToHost, ctx->stream));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int fmvs_apply_mask(fmvs_ctx* ctx, float* depth, float* normals_xyz, float* confidence, int32_t w,
                    int32_t h, const uint8_t* mask) {
    return guarded([&] {
        ctx->use();
        const size_t px = static_cast<size_t>(std::max(w, 0)) * std::max(h, 0);
        if (!px)
            return;
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        float* d = t.upload(depth, px, s);
        float* n = t.upload(normals_xyz, 3 * px, s);
        float* c = t.upload(confidence, px, s);
        const uint8_t* m = t.upload(mask, px, s);
        k::apply_mask(d, n, c, m, static_cast<int>(px), s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(depth, d, px * 4, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaMemcpyAsync(normals_xyz, n, 3 * px * 4, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaMemcpyAsync(confidence, c, px * 4, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

void fmvs_geom_filter_config_default(fmvs_geom_filter_config* c) {
    c->eta_r = 10.0;  // postfilter.hpp:32-36
    c->eta_h = 3;
    c->lookup = FMVS_LOOKUP_NEAREST;
}

int fmvs_geometric_consistency_mask(fmvs_ctx* ctx, const fmvs_consistency_view* window, int32_t n,
                                    int32_t ref_index, const fmvs_geom_filter_config* cfg,
                                    uint8_t* keep) {
    return guarded([&] {
        ctx->use();
        fmvs_geom_filter_config c;
        fmvs_geom_filter_config_default(&c);
        if (cfg)
            c = *cfg;
        check_geom_window(n, ref_index, c);
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        std::vector<k::GeomView> gv(n);
        for (int i = 0; i < n; ++i) {
            const size_t px = static_cast<size_t>(window[i].width) * window[i].height;
            gv[i] = geom_view(t.upload(window[i].depth, px, s), window[i].width, window[i].height,
                              window[i].intrinsics, window[i].pose);
        }
        const int w = window[ref_index].width, h = window[ref_index].height;
        const size_t px = static_cast<size_t>(std::max(w, 0)) * std::max(h, 0);
        if (!px)
            return;
        k::GeomArgs ga{};
        ga.views = t.upload(gv.data(), gv.size(), s);
        ga.n = n;
        ga.ref = ref_index;
        ga.eta_r = c.eta_r;
        ga.eta_h = c.eta_h;
        ga.bilinear = c.lookup == FMVS_LOOKUP_BILINEAR;
        ga.keep = t.alloc<uint8_t>(px);
        k::geometric_mask(ga, w, h, s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(keep, ga.keep, px, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int fmvs_estimate_sequence(fmvs_ctx* ctx, const fmvs_view* frames, int32_t n_frames, int32_t stride,
                           const fmvs_config* cfg, int32_t filter, float* depth, float* normals_xyz,
                           float* confidence, int32_t* ref_frames, int32_t capacity,
                           int32_t* n_results) {
    if (n_results)
        *n_results = 0;
    return guarded([&] {
        ctx->use();
        if (!cfg)
            fmvs::fail_config("estimate: null config");
        // tools/fassmvs.cpp:93-119 (CLI checks, then PipelineConfig::validate)
        if (cfg->bundle_size < 3 || cfg->bundle_size % 2 == 0)
            fmvs::fail_config("--bundle-size must be odd and at least 3");
        if (stride < 1)
            fmvs::fail_config("--stride must be at least 1");
        if (filter < FMVS_FILTER_NONE || filter > FMVS_FILTER_BOTH)
            fmvs::fail_config("--filter must be none, dog, geom or both");
        fmvs::validate_config(*cfg);
        for (int i = 0; i < n_frames; ++i)  // :121-133
            fmvs::validate_view(frames[i]);
        if (n_frames < cfg->bundle_size)  // :134-135
            fmvs::fail_input("sequence shorter than one bundle");
        const int half = cfg->bundle_size / 2;
        std::vector<int> refs;  // :145-149
        for (int r = half; r + half < n_frames; r += stride)
            refs.push_back(r);
        const int m = static_cast<int>(refs.size());
        if (n_results)
            *n_results = m;
        if (m > capacity)
            throw fmvs::Error(FMVS_ERR_CAPACITY, "estimate_sequence: result capacity too small");
        const int w = frames[0].intrinsics.width, h = frames[0].intrinsics.height;
        for (int i = 0; i < n_frames; ++i)
            if (frames[i].intrinsics.width != w || frames[i].intrinsics.height != h)
                fmvs::fail_input("estimate_sequence: frames must share one size");
        const size_t px = static_cast<size_t>(w) * h;
        cudaStream_t s = ctx->stream;
        // frames resident on the device once; bundles reference them in place
        uint8_t* d_frames = ctx->buf("seq_frames").as<uint8_t>(px * n_frames);
        for (int i = 0; i < n_frames; ++i)
            FMVS_CUDA_CHECK(cudaMemcpyAsync(d_frames + i * px, frames[i].image, px, cudaMemcpyHostToDevice, s));
        float* d_maps = ctx->buf("seq_maps").as<float>(5 * px * m);  // depth | normals | conf
        float* d_depth = d_maps;
        float* d_normals = d_maps + px * m;
        float* d_conf = d_maps + 4 * px * m;
        std::vector<const uint8_t*> d_images(cfg->bundle_size);
        for (int r = 0; r < m; ++r) {
            const int first = refs[r] - half;
            for (int k2 = 0; k2 < cfg->bundle_size; ++k2)
                d_images[k2] = d_frames + (first + k2) * px;
            run_bundle(ctx, frames + first, cfg->bundle_size, *cfg, d_images.data(), d_depth + r * px,
                       d_normals + 3 * r * px, d_conf + r * px);
        }
        uint8_t* d_mask = ctx->buf("seq_masks").as<uint8_t>(px * std::max(m, 1));
        if (filter == FMVS_FILTER_DOG || filter == FMVS_FILTER_BOTH) {  // :151-158
            for (int r = 0; r < m; ++r) {
                dog_mask_device(ctx, d_frames + refs[r] * px, w, h, d_mask);
                k::apply_mask(d_depth + r * px, d_normals + 3 * r * px, d_conf + r * px, d_mask,
                              static_cast<int>(px), s);
            }
        }
        if (filter == FMVS_FILTER_GEOM || filter == FMVS_FILTER_BOTH) {  // :159-176
            fmvs_geom_filter_config gc;
            fmvs_geom_filter_config_default(&gc);
            const int ws = std::min(5, m);
            check_geom_window(ws, 0, gc);
            std::vector<k::GeomView> gv(m);
            for (int r = 0; r < m; ++r)
                gv[r] = geom_view(d_depth + r * px, w, h, frames[refs[r]].intrinsics, frames[refs[r]].pose);
            k::GeomView* d_gv = ctx->buf("seq_geom_views").as<k::GeomView>(m);
            FMVS_CUDA_CHECK(cudaMemcpyAsync(d_gv, gv.data(), sizeof(k::GeomView) * m, cudaMemcpyHostToDevice, s));
            // every mask from the unfiltered window before any is applied
            for (int i = 0; i < m; ++i) {
                const int start = std::clamp(i - ws / 2, 0, m - ws);
                k::GeomArgs ga{};
                ga.views = d_gv + start;
                ga.n = ws;
                ga.ref = i - start;
                ga.eta_r = gc.eta_r;
                ga.eta_h = gc.eta_h;
                ga.bilinear = gc.lookup == FMVS_LOOKUP_BILINEAR;
                ga.keep = d_mask + i * px;
                k::geometric_mask(ga, w, h, s);
            }
            for (int i = 0; i < m; ++i)
                k::apply_mask(d_depth + i * px, d_normals + 3 * i * px, d_conf + i * px, d_mask + i * px,
                              static_cast<int>(px), s);
        }
        FMVS_CUDA_CHECK(cudaMemcpyAsync(depth, d_depth, 4 * px * m, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaMemcpyAsync(normals_xyz, d_normals, 12 * px * m, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaMemcpyAsync(confidence, d_conf, 4 * px * m, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
        for (int r = 0; r < m; ++r)
            ref_frames[r] = refs[r];
        finish_stats(ctx);
        ctx->collect();
    });
}

}  // extern "C"

// ======================================================= multi-GPU sequence
// fmvs_estimate_sequence_multi: the `fassmvs estimate` loop (tools/fassmvs.cpp:
// 139-176) sharded over GPUs. Results (bundles) are independent
// (SPEC.md:408), so each device owns a contiguous shard and runs it with
// `inflight` bundles in flight (one context = one stream each). Post-filters
// run on a per-device post stream as soon as their inputs exist; results
// stream back to the caller's buffers one by one (D2H right after the result
// is final), and device memory is a bounded pool of result slots. The only
// cross-device data is the geometric filter's window (postfilter.cpp:95-160):
// the DoG-filtered depth maps of the few results at shard boundaries, copied
// peer to peer (cudaMemcpyPeerAsync over NVLink) after the producer's event.

namespace {

// Window of the geometric filter for result i of m (ws = min(5, m);
// tools/fassmvs.cpp:163-172): [start, start + ws).
int window_start(int i, int m, int ws) { return std::clamp(i - ws / 2, 0, m - ws); }

struct SeqPlan {
    std::vector<int> begin, end;  // shard bounds over results
    // per shard: results imported from other shards / exported to them
    std::vector<std::vector<int>> imports, exports;
};

SeqPlan plan_sequence(int m, int shards, int ws) {
    SeqPlan p;
    p.begin.resize(shards);
    p.end.resize(shards);
    const int base = m / shards, extra = m % shards;
    int at = 0;
    for (int s = 0; s < shards; ++s) {
        p.begin[s] = at;
        at += base + (s < extra ? 1 : 0);
        p.end[s] = at;
    }
    p.imports.assign(shards, {});
    p.exports.assign(shards, {});
    if (ws <= 1)
        return p;
    std::vector<int> owner(m);
    for (int s = 0; s < shards; ++s)
        for (int k = p.begin[s]; k < p.end[s]; ++k)
            owner[k] = s;
    std::vector<std::vector<char>> need(shards, std::vector<char>(m, 0));
    for (int s = 0; s < shards; ++s)
        for (int i = p.begin[s]; i < p.end[s]; ++i) {
            const int st = window_start(i, m, ws);
            for (int k = st; k < st + ws; ++k)
                if (owner[k] != s)
                    need[s][k] = 1;
        }
    std::vector<char> exported(m, 0);
    for (int s = 0; s < shards; ++s)
        for (int k = 0; k < m; ++k)
            if (need[s][k]) {
                p.imports[s].push_back(k);
                exported[k] = 1;
            }
    for (int k = 0; k < m; ++k)
        if (exported[k])
            p.exports[owner[k]].push_back(k);
    return p;
}

// Host-side publication of exported (DoG-filtered) depth maps.
struct HaloBoard {
    std::mutex mu;
    std::condition_variable cv;
    struct Entry {
        const float* depth = nullptr;
        int device = 0;
        cudaEvent_t ready = nullptr;
    };
    std::unordered_map<int, Entry> posted;
    bool failed = false;

    void post(int k, const Entry& e) {
        {
            std::lock_guard<std::mutex> g(mu);
            posted[k] = e;
        }
        cv.notify_all();
    }
    // false when another shard failed (the caller then stops)
    bool wait(int k, Entry* out) {
        std::unique_lock<std::mutex> g(mu);
        cv.wait(g, [&] { return failed || posted.count(k) > 0; });
        if (failed)
            return false;
        *out = posted[k];
        return true;
    }
    void fail() {
        {
            std::lock_guard<std::mutex> g(mu);
            failed = true;
        }
        cv.notify_all();
    }
};

struct SeqJob {
    const fmvs_view* frames;
    int n_frames;
    const fmvs_config* cfg;
    int filter;
    int m, ws, half, w, h;
    std::vector<int> refs;
    float* depth;
    float* normals;
    float* conf;
    fmvs_geom_filter_config gc;
};

bool host_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// One shard on one device: everything its host thread owns.
struct Shard {
    int device = 0, begin = 0, end = 0, inflight = 1;
    std::vector<int> imports, exports;
    std::vector<fmvs_ctx*> ctxs;
    fmvs_ctx* post = nullptr;  // its stream is the post stream; its buffers hold masks
    std::vector<void*> allocs;
    std::vector<cudaEvent_t> events;
    std::string error;
    int code = FMVS_OK;

    float* alloc_maps(size_t px) {
        void* p = nullptr;
        FMVS_CUDA_CHECK(cudaMalloc(&p, 5 * px * sizeof(float)));
        allocs.push_back(p);
        return static_cast<float*>(p);
    }
    cudaEvent_t event() {
        cudaEvent_t e;
        FMVS_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        events.push_back(e);
        return e;
    }
    void release() {
        FMVS_CUDA_CHECK(cudaSetDevice(device));
        for (void* p : allocs)
            cudaFree(p);
        for (cudaEvent_t e : events)
            cudaEventDestroy(e);
        for (fmvs_ctx* c : ctxs)
            fmvs_ctx_destroy(c);
        if (post)
            fmvs_ctx_destroy(post);
        allocs.clear();
        events.clear();
        ctxs.clear();
        post = nullptr;
    }
};

void run_shard(Shard& sh, const SeqJob& job, HaloBoard& board) {
    FMVS_CUDA_CHECK(cudaSetDevice(sh.device));
    const size_t px = static_cast<size_t>(job.w) * job.h;
    const int nb = job.cfg->bundle_size;
    for (int i = 0; i < sh.inflight; ++i) {
        fmvs_ctx* c = nullptr;
        const int rc = fmvs_ctx_create(sh.device, &c);
        if (rc != FMVS_OK)
            throw Error(rc, g_last_error);
        sh.ctxs.push_back(c);
    }
    {
        fmvs_ctx* c = nullptr;
        const int rc = fmvs_ctx_create(sh.device, &c);
        if (rc != FMVS_OK)
            throw Error(rc, g_last_error);
        sh.post = c;
    }
    cudaStream_t ps = sh.post->stream;
    if (sh.begin >= sh.end)
        return;

    // frames of this shard, resident once; bundles reference them in place
    const int f0 = job.refs[sh.begin] - job.half;
    const int f1 = job.refs[sh.end - 1] + job.half + 1;
    uint8_t* d_frames = sh.post->buf("seq_frames").as<uint8_t>(px * (f1 - f0));
    for (int f = f0; f < f1; ++f)
        FMVS_CUDA_CHECK(cudaMemcpyAsync(d_frames + (f - f0) * px, job.frames[f].image, px,
                                        cudaMemcpyHostToDevice, ps));
    cudaEvent_t frames_ready = sh.event();
    FMVS_CUDA_CHECK(cudaEventRecord(frames_ready, ps));
    for (fmvs_ctx* c : sh.ctxs)
        FMVS_CUDA_CHECK(cudaStreamWaitEvent(c->stream, frames_ready, 0));

    const bool dog = job.filter == FMVS_FILTER_DOG || job.filter == FMVS_FILTER_BOTH;
    const bool geom = job.ws > 1;
    const int m = job.m;
    // last post step (result index) that reads result k
    auto last_user = [&](int k) {
        int last = k;
        if (geom)
            for (int i = std::max(0, k - job.ws + 1); i < std::min(m, k + job.ws); ++i) {
                const int st = window_start(i, m, job.ws);
                if (k >= st && k < st + job.ws)
                    last = std::max(last, i);
            }
        return last;
    };

    // result slots: depth | normals | conf (5 px floats). Exported results
    // keep theirs to the end; the others cycle through a pool, a slot going
    // back to the pool after the post step of its last reader (recorded on
    // the post stream; the next bundle in it waits for that event).
    struct PoolSlot {
        float* maps;
        cudaEvent_t after;
    };
    std::vector<PoolSlot> pool;  // FIFO: the longest-released slot is reused first
    size_t pool_head = 0;
    int pooled_slots = 0;
    // enough slots that `inflight` bundles never wait for each other's D2H
    const int min_slots = sh.inflight + job.ws + 2;
    std::unordered_map<int, float*> slot_of;  // result -> maps (local and imported)
    std::vector<std::pair<int, int>> held;    // (last reader, result) of pooled slots in use
    const std::vector<int>& ex = sh.exports;
    auto is_export = [&](int k) { return std::binary_search(ex.begin(), ex.end(), k); };

    uint8_t* dog_mask = sh.post->buf("seq_dog").as<uint8_t>(px);
    uint8_t* keep = sh.post->buf("seq_keep").as<uint8_t>(px);
    float* out_depth = sh.post->buf("seq_out_depth").as<float>(px);
    const int nlocal = sh.end - sh.begin;
    k::GeomView* gv_host = nullptr;
    k::GeomView* gv_dev = nullptr;
    HostBuf gv_pinned;
    if (geom) {
        gv_host = static_cast<k::GeomView*>(gv_pinned.get(sizeof(k::GeomView) * nlocal * job.ws));
        gv_dev = sh.post->buf("seq_geom_views").as<k::GeomView>(static_cast<size_t>(nlocal) * job.ws);
    }
    // D2H: straight into the caller's buffers when they are pinned, else
    // through pinned staging slots drained by this thread
    const bool direct = host_pinned(job.depth) && host_pinned(job.normals) && host_pinned(job.conf);
    struct Staged {
        int k;
        float* host;
        cudaEvent_t done;
    };
    std::vector<Staged> staged;  // in flight
    std::vector<std::pair<float*, cudaEvent_t>> stage_free;
    auto drain = [&](bool all) {
        while (!staged.empty()) {
            Staged& st = staged.front();
            if (!all && cudaEventQuery(st.done) == cudaErrorNotReady) {
                cudaGetLastError();
                break;
            }
            FMVS_CUDA_CHECK(cudaEventSynchronize(st.done));
            std::memcpy(job.depth + st.k * px, st.host, 4 * px);
            std::memcpy(job.normals + 3 * st.k * px, st.host + px, 12 * px);
            std::memcpy(job.conf + st.k * px, st.host + 4 * px, 4 * px);
            stage_free.push_back({st.host, st.done});
            staged.erase(staged.begin());
        }
    };
    HostBuf stage_mem;  // pinned staging ring (grown to 2 * inflight + 2 slots)
    std::vector<float*> stage_slots;

    // bundle order: exported results first (so every shard publishes its
    // halo before it could wait for another's), then the rest ascending
    std::vector<int> order(ex.begin(), ex.end());
    for (int k = sh.begin; k < sh.end; ++k)
        if (!is_export(k))
            order.push_back(k);
    std::vector<char> enqueued(m, 0);
    int next_post = sh.begin;
    int rr = 0;

    auto post_step = [&](int i) {
        float* mi = slot_of.at(i);
        float* dep = mi;
        float* nrm = mi + px;
        float* cf = mi + 4 * px;
        const float* final_depth = dep;
        if (geom) {
            const int st = window_start(i, m, job.ws);
            for (int j = 0; j < job.ws; ++j) {
                const int kk = st + j;
                if (!slot_of.count(kk)) {  // import from the owning shard
                    HaloBoard::Entry e;
                    if (!board.wait(kk, &e))
                        throw Error(FMVS_ERR_CUDA, "sequence: another shard failed");
                    float* dst = sh.alloc_maps(px);  // depth only is used
                    FMVS_CUDA_CHECK(cudaStreamWaitEvent(ps, e.ready, 0));
                    FMVS_CUDA_CHECK(cudaMemcpyPeerAsync(dst, sh.device, e.depth, e.device, 4 * px, ps));
                    slot_of[kk] = dst;
                }
                const int fr = job.refs[kk];
                gv_host[(i - sh.begin) * job.ws + j] =
                    geom_view(slot_of[kk], job.w, job.h, job.frames[fr].intrinsics, job.frames[fr].pose);
            }
            k::GeomView* g = gv_dev + static_cast<size_t>(i - sh.begin) * job.ws;
            FMVS_CUDA_CHECK(cudaMemcpyAsync(g, gv_host + (i - sh.begin) * job.ws, sizeof(k::GeomView) * job.ws,
                                            cudaMemcpyHostToDevice, ps));
            k::GeomArgs ga{};
            ga.views = g;
            ga.n = job.ws;
            ga.ref = i - st;
            ga.eta_r = job.gc.eta_r;
            ga.eta_h = job.gc.eta_h;
            ga.bilinear = job.gc.lookup == FMVS_LOOKUP_BILINEAR;
            ga.keep = keep;
            k::geometric_mask(ga, job.w, job.h, ps);
            // the slot keeps the DoG-filtered depth for later windows; the
            // final depth is a masked copy
            FMVS_CUDA_CHECK(cudaMemcpyAsync(out_depth, dep, 4 * px, cudaMemcpyDeviceToDevice, ps));
            k::apply_mask(out_depth, nrm, cf, keep, static_cast<int>(px), ps);
            final_depth = out_depth;
        }
        if (direct) {
            FMVS_CUDA_CHECK(cudaMemcpyAsync(job.depth + i * px, final_depth, 4 * px, cudaMemcpyDeviceToHost, ps));
            FMVS_CUDA_CHECK(cudaMemcpyAsync(job.normals + 3 * i * px, nrm, 12 * px, cudaMemcpyDeviceToHost, ps));
            FMVS_CUDA_CHECK(cudaMemcpyAsync(job.conf + i * px, cf, 4 * px, cudaMemcpyDeviceToHost, ps));
        } else {
            drain(false);
            float* hs = nullptr;
            cudaEvent_t done = nullptr;
            if (!stage_free.empty()) {
                hs = stage_free.back().first;
                done = stage_free.back().second;
                stage_free.pop_back();
            } else if (stage_slots.size() < static_cast<size_t>(2 * sh.inflight + 2)) {
                if (stage_slots.empty())
                    stage_mem.get(sizeof(float) * 5 * px * (2 * sh.inflight + 2));
                hs = static_cast<float*>(stage_mem.ptr) + 5 * px * stage_slots.size();
                stage_slots.push_back(hs);
                done = sh.event();
            } else {
                drain(true);
                hs = stage_free.back().first;
                done = stage_free.back().second;
                stage_free.pop_back();
            }
            FMVS_CUDA_CHECK(cudaMemcpyAsync(hs, final_depth, 4 * px, cudaMemcpyDeviceToHost, ps));
            FMVS_CUDA_CHECK(cudaMemcpyAsync(hs + px, nrm, 12 * px, cudaMemcpyDeviceToHost, ps));
            FMVS_CUDA_CHECK(cudaMemcpyAsync(hs + 4 * px, cf, 4 * px, cudaMemcpyDeviceToHost, ps));
            FMVS_CUDA_CHECK(cudaEventRecord(done, ps));
            staged.push_back({i, hs, done});
        }
        // release pooled slots whose last reader was this step
        cudaEvent_t after = nullptr;
        for (auto it = held.begin(); it != held.end();) {
            if (it->first <= i) {
                if (!after) {
                    after = sh.event();
                    FMVS_CUDA_CHECK(cudaEventRecord(after, ps));
                }
                pool.push_back({slot_of[it->second], after});
                it = held.erase(it);
            } else {
                ++it;
            }
        }
    };

    for (size_t pos = 0; pos < order.size(); ++pos) {
        const int k = order[pos];
        fmvs_ctx* c = sh.ctxs[rr++ % sh.inflight];
        float* maps = nullptr;
        if (is_export(k)) {
            maps = sh.alloc_maps(px);
        } else {
            if (pool_head < pool.size() && pooled_slots >= min_slots) {
                maps = pool[pool_head].maps;
                FMVS_CUDA_CHECK(cudaStreamWaitEvent(c->stream, pool[pool_head].after, 0));
                ++pool_head;
            } else {
                maps = sh.alloc_maps(px);
                ++pooled_slots;
            }
            held.push_back({last_user(k), k});
        }
        slot_of[k] = maps;
        const int first = job.refs[k] - job.half;
        std::vector<const uint8_t*> d_images(nb);
        for (int v = 0; v < nb; ++v)
            d_images[v] = d_frames + (first + v - f0) * px;
        run_bundle(c, job.frames + first, nb, *job.cfg, d_images.data(), maps, maps + px, maps + 4 * px);
        cudaEvent_t done = sh.event();
        FMVS_CUDA_CHECK(cudaEventRecord(done, c->stream));
        FMVS_CUDA_CHECK(cudaStreamWaitEvent(ps, done, 0));
        if (dog) {  // tools/fassmvs.cpp:151-158
            dog_mask_device(sh.post, d_frames + (job.refs[k] - f0) * px, job.w, job.h, dog_mask);
            k::apply_mask(maps, maps + px, maps + 4 * px, dog_mask, static_cast<int>(px), ps);
        }
        if (is_export(k)) {
            cudaEvent_t ready = sh.event();
            FMVS_CUDA_CHECK(cudaEventRecord(ready, ps));
            board.post(k, HaloBoard::Entry{maps, sh.device, ready});
        }
        enqueued[k] = 1;
        // every result whose window is now enqueued locally (imports are
        // awaited inside the step). Not before all exports are posted: a
        // shard never waits for another while holding back its own halo.
        if (pos + 1 < ex.size())
            continue;
        while (next_post < sh.end) {
            bool ready = true;
            if (geom) {
                const int st = window_start(next_post, m, job.ws);
                for (int kk = st; kk < st + job.ws; ++kk)
                    if (kk >= sh.begin && kk < sh.end && !enqueued[kk])
                        ready = false;
            } else {
                ready = enqueued[next_post] != 0;
            }
            if (!ready)
                break;
            post_step(next_post++);
        }
    }
    FMVS_CUDA_CHECK(cudaStreamSynchronize(ps));
    for (fmvs_ctx* c : sh.ctxs)
        FMVS_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    drain(true);
}

}  // namespace

extern "C" {

int fmvs_sequence_plan(int32_t m, int32_t n_shards, int32_t shard, int32_t window, int32_t* begin,
                       int32_t* end, int32_t* imports, int32_t* n_imports, int32_t* exports,
                       int32_t* n_exports) {
    return guarded([&] {
        if (m < 0 || n_shards < 1 || shard < 0 || shard >= n_shards || window < 0 || window > std::max(m, 0))
            fmvs::fail_input("sequence plan: invalid arguments");
        const SeqPlan p = plan_sequence(m, n_shards, window);
        *begin = p.begin[shard];
        *end = p.end[shard];
        *n_imports = static_cast<int32_t>(p.imports[shard].size());
        *n_exports = static_cast<int32_t>(p.exports[shard].size());
        if (imports)
            std::copy(p.imports[shard].begin(), p.imports[shard].end(), imports);
        if (exports)
            std::copy(p.exports[shard].begin(), p.exports[shard].end(), exports);
    });
}

int fmvs_estimate_sequence_multi(const int32_t* devices, int32_t n_devices, int32_t inflight,
                                 const fmvs_view* frames, int32_t n_frames, int32_t stride,
                                 const fmvs_config* cfg, int32_t filter, float* depth, float* normals_xyz,
                                 float* confidence, int32_t* ref_frames, int32_t capacity,
                                 int32_t* n_results) {
    if (n_results)
        *n_results = 0;
    std::vector<Shard> shards;
    int rc = guarded([&] {
        if (!devices || n_devices < 1)
            fmvs::fail_input("sequence: no devices");
        if (inflight < 1)
            fmvs::fail_config("sequence: inflight must be at least 1");
        if (!cfg)
            fmvs::fail_config("estimate: null config");
        // the CLI's checks, in its order (tools/fassmvs.cpp:93-135)
        if (cfg->bundle_size < 3 || cfg->bundle_size % 2 == 0)
            fmvs::fail_config("--bundle-size must be odd and at least 3");
        if (stride < 1)
            fmvs::fail_config("--stride must be at least 1");
        if (filter < FMVS_FILTER_NONE || filter > FMVS_FILTER_BOTH)
            fmvs::fail_config("--filter must be none, dog, geom or both");
        fmvs::validate_config(*cfg);
        for (int i = 0; i < n_frames; ++i)
            fmvs::validate_view(frames[i]);
        if (n_frames < cfg->bundle_size)
            fmvs::fail_input("sequence shorter than one bundle");
        SeqJob job{};
        job.frames = frames;
        job.n_frames = n_frames;
        job.cfg = cfg;
        job.filter = filter;
        job.half = cfg->bundle_size / 2;
        for (int r = job.half; r + job.half < n_frames; r += stride)
            job.refs.push_back(r);
        job.m = static_cast<int>(job.refs.size());
        if (n_results)
            *n_results = job.m;
        if (job.m > capacity)
            throw Error(FMVS_ERR_CAPACITY, "estimate_sequence: result capacity too small");
        job.w = frames[0].intrinsics.width;
        job.h = frames[0].intrinsics.height;
        for (int i = 0; i < n_frames; ++i)
            if (frames[i].intrinsics.width != job.w || frames[i].intrinsics.height != job.h)
                fmvs::fail_input("estimate_sequence: frames must share one size");
        fmvs_geom_filter_config_default(&job.gc);
        job.ws = 0;
        if (filter == FMVS_FILTER_GEOM || filter == FMVS_FILTER_BOTH) {
            job.ws = std::min(5, job.m);
            check_geom_window(job.ws, 0, job.gc);
        }
        job.depth = depth;
        job.normals = normals_xyz;
        job.conf = confidence;
        const SeqPlan plan = plan_sequence(job.m, n_devices, job.ws);
        shards.resize(n_devices);
        for (int d = 0; d < n_devices; ++d) {
            shards[d].device = devices[d];
            shards[d].begin = plan.begin[d];
            shards[d].end = plan.end[d];
            shards[d].inflight = inflight;
            shards[d].imports = plan.imports[d];
            shards[d].exports = plan.exports[d];
        }
        // NVLink peer access between devices that exchange halos
        for (int d = 0; d < n_devices; ++d)
            for (int e = 0; e < n_devices; ++e) {
                if (devices[d] == devices[e] || shards[d].imports.empty())
                    continue;
                int can = 0;
                if (cudaDeviceCanAccessPeer(&can, devices[d], devices[e]) == cudaSuccess && can) {
                    FMVS_CUDA_CHECK(cudaSetDevice(devices[d]));
                    const cudaError_t pe = cudaDeviceEnablePeerAccess(devices[e], 0);
                    if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
                        FMVS_CUDA_CHECK(pe);
                    cudaGetLastError();
                }
            }
        HaloBoard board;
        std::vector<std::thread> threads;
        for (int d = 0; d < n_devices; ++d)
            threads.emplace_back([&, d] {
                Shard& sh = shards[d];
                sh.code = guarded([&] { run_shard(sh, job, board); });
                if (sh.code != FMVS_OK) {
                    sh.error = g_last_error;
                    board.fail();
                }
            });
        for (auto& t : threads)
            t.join();
        for (const Shard& sh : shards)
            if (sh.code != FMVS_OK)
                throw Error(sh.code, sh.error);
        for (int r = 0; r < job.m; ++r)
            ref_frames[r] = job.refs[r];
    });
    // every shard's streams are idle here (joined; on failure, synchronise
    // before freeing: peers may still read exported buffers)
    for (Shard& sh : shards) {
        cudaSetDevice(sh.device);
        cudaDeviceSynchronize();
    }
    for (Shard& sh : shards)
        sh.release();
    return rc;
}
}  // extern "C"

// ------------------------------------------------ output stage (§8f) --
extern "C" {

namespace {
int colorize_host(fmvs_ctx* ctx, int kind, const float* in, int w, int h, double lo, double hi,
                  uint8_t* rgb) {
    return guarded([&] {
        ctx->use();
        const size_t px = static_cast<size_t>(std::max(w, 0)) * std::max(h, 0);
        if (!px)
            return;
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const float* d_in = t.upload(in, px * (kind == 1 ? 3 : 1), s);
        uint8_t* d_rgb = t.alloc<uint8_t>(3 * px);
        k::colorize(kind, d_in, static_cast<int>(px), lo, hi, d_rgb, s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(rgb, d_rgb, 3 * px, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}
}  // namespace

int fmvs_colorize_depth(fmvs_ctx* ctx, const float* depth, int32_t w, int32_t h, double lo, double hi,
                        uint8_t* rgb) {
    return colorize_host(ctx, 0, depth, w, h, lo, hi, rgb);
}

int fmvs_colorize_normals(fmvs_ctx* ctx, const float* normals_xyz, int32_t w, int32_t h, uint8_t* rgb) {
    return colorize_host(ctx, 1, normals_xyz, w, h, 0.0, 0.0, rgb);
}

int fmvs_colorize_confidence(fmvs_ctx* ctx, const float* conf, int32_t w, int32_t h, uint8_t* rgb) {
    return colorize_host(ctx, 2, conf, w, h, 0.0, 0.0, rgb);
}

int fmvs_write_pfm(const char* path, const float* data, int32_t w, int32_t h, int32_t channels) {
    return guarded([&] {
        if (channels != 1 && channels != 3)
            fmvs::fail_input("write_pfm: channels must be 1 or 3");
        std::FILE* f = std::fopen(path, "wb");
        if (!f)
            fmvs::fail_input(std::string("cannot open for writing: ") + path);  // map_io.cpp:20-25
        const std::string hdr = std::string(channels == 1 ? "Pf" : "PF") + "\n" + std::to_string(w) +
                                " " + std::to_string(h) + "\n-1.0\n";
        bool ok = std::fwrite(hdr.data(), 1, hdr.size(), f) == hdr.size();
        const size_t row = static_cast<size_t>(w) * channels;
        for (int y = h - 1; y >= 0 && ok; --y)  // bottom-to-top rows
            ok = std::fwrite(data + static_cast<size_t>(y) * row, sizeof(float), row, f) == row;
        ok = (std::fclose(f) == 0) && ok;
        if (!ok)
            fmvs::fail_input("short write on float map file");
    });
}

// write_png (map_io.cpp:203-260): signature, IHDR (8-bit RGB), one IDAT of
// the filter-0 scanlines deflated by compress2 at level 6, IEND; every chunk
// is length (big endian), type, data, CRC-32 over type + data.
int fmvs_write_png(const char* path, const uint8_t* rgb, int32_t w, int32_t h) {
    return guarded([&] {
        std::FILE* f = std::fopen(path, "wb");
        if (!f)
            fmvs::fail_input(std::string("cannot open for writing: ") + path);  // map_io.cpp:20-25
        std::vector<uint8_t> out;
        auto be32 = [&](uint32_t v) {
            const uint8_t b[4] = {uint8_t(v >> 24), uint8_t(v >> 16), uint8_t(v >> 8), uint8_t(v)};
            out.insert(out.end(), b, b + 4);
        };
        auto chunk = [&](const char* type, const uint8_t* data, size_t n) {
            be32(static_cast<uint32_t>(n));
            out.insert(out.end(), type, type + 4);
            if (n)
                out.insert(out.end(), data, data + n);
            uLong crc = crc32(0L, reinterpret_cast<const Bytef*>(type), 4);
            if (n)
                crc = crc32(crc, data, static_cast<uInt>(n));
            be32(static_cast<uint32_t>(crc));
        };
        static const uint8_t sig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};
        out.insert(out.end(), sig, sig + 8);
        uint8_t ihdr[13] = {0};
        const uint32_t uw = static_cast<uint32_t>(w), uh = static_cast<uint32_t>(h);
        for (int i = 0; i < 4; ++i) {
            ihdr[i] = static_cast<uint8_t>(uw >> (24 - 8 * i));
            ihdr[4 + i] = static_cast<uint8_t>(uh >> (24 - 8 * i));
        }
        ihdr[8] = 8;  // bit depth
        ihdr[9] = 2;  // RGB
        chunk("IHDR", ihdr, 13);
        const size_t row = 3 * static_cast<size_t>(w > 0 ? w : 0);
        std::vector<uint8_t> raw;
        raw.reserve(static_cast<size_t>(h > 0 ? h : 0) * (1 + row));
        for (int y = 0; y < h; ++y) {
            raw.push_back(0);  // filter type 0 per scanline
            raw.insert(raw.end(), rgb + static_cast<size_t>(y) * row, rgb + static_cast<size_t>(y + 1) * row);
        }
        uLongf bound = compressBound(static_cast<uLong>(raw.size()));
        std::vector<uint8_t> z(bound);
        if (compress2(z.data(), &bound, raw.data(), static_cast<uLong>(raw.size()), 6) != Z_OK) {
            std::fclose(f);
            fmvs::fail_input(std::string("png compression failed: ") + path);
        }
        chunk("IDAT", z.data(), bound);
        chunk("IEND", nullptr, 0);
        bool ok = std::fwrite(out.data(), 1, out.size(), f) == out.size();
        ok = (std::fclose(f) == 0) && ok;
        if (!ok)
            fmvs::fail_input(std::string("short write: ") + path);
    });
}

}  // extern "C"

// ------------------------------------------- accuracy scoring (§8f) --
extern "C" {

int fmvs_evaluate(fmvs_ctx* ctx, const float* est, const float* gt, int32_t w, int32_t h,
                  const double* thetas, int32_t n_thetas, fmvs_l1_result* l1, fmvs_acc_cpl_f* scores) {
    return guarded([&] {
        ctx->use();
        if (w <= 0 || h <= 0)
            fmvs::fail_input("metrics: maps must be non-empty and equal size");  // evaluation.cpp:17-20
        if (n_thetas < 0 || n_thetas > 16)
            fmvs::fail_input("evaluate: at most 16 thresholds");
        const size_t px = static_cast<size_t>(w) * h;
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const float* d_est = t.upload(est, px, s);
        const float* d_gt = t.upload(gt, px, s);
        k::EvalThetas th{};
        th.n = n_thetas;
        for (int i = 0; i < n_thetas; ++i)
            th.theta[i] = thetas[i];
        auto* counts = t.alloc<unsigned long long>(3 + 16);
        const size_t nb = (px + 255) / 256;
        auto* partials = t.alloc<double>(2 * nb);
        auto* sums = t.alloc<double>(2);
        k::evaluate_counts(d_est, d_gt, static_cast<int>(px), th, counts, partials, sums, s);
        unsigned long long hc[19] = {};
        double hs[2] = {};
        FMVS_CUDA_CHECK(cudaMemcpyAsync(hc, counts, sizeof(unsigned long long) * (3 + n_thetas),
                                        cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaMemcpyAsync(hs, sums, sizeof(hs), cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
        const unsigned long long valid_est = hc[0], valid_gt = hc[1], both = hc[2];
        if (both == 0)
            fmvs::fail_input("metrics: no pixel is valid in both maps");
        l1->valid_both = both;
        l1->l1_abs = hs[0] / static_cast<double>(both);
        l1->l1_rel = hs[1] / static_cast<double>(both);
        for (int i = 0; i < n_thetas; ++i) {  // evaluation.cpp:67-70
            fmvs_acc_cpl_f& r = scores[i];
            const unsigned long long pass = hc[3 + i];
            r.valid_both = both;
            r.valid_est = valid_est;
            r.valid_gt = valid_gt;
            r.acc = valid_est ? static_cast<double>(pass) / valid_est : 0.0;
            r.cpl = valid_gt ? static_cast<double>(pass) / valid_gt : 0.0;
            r.f = (r.acc + r.cpl) > 0.0 ? 2.0 * r.acc * r.cpl / (r.acc + r.cpl) : 0.0;
        }
    });
}

int fmvs_roc_curve(fmvs_ctx* ctx, const float* est, const float* gt, const float* conf, int32_t w,
                   int32_t h, double theta, double* densities, double* error_rates) {
    return guarded([&] {
        ctx->use();
        if (w <= 0 || h <= 0)
            fmvs::fail_input("metrics: maps must be non-empty and equal size");
        const size_t px = static_cast<size_t>(w) * h;
        const int n = static_cast<int>(px);
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const float* d_est = t.upload(est, px, s);
        const float* d_gt = t.upload(gt, px, s);
        const float* d_conf = t.upload(conf, px, s);
        float* keys = t.alloc<float>(px);
        float* keys_sorted = t.alloc<float>(px);
        uint8_t* pass = t.alloc<uint8_t>(px);
        uint8_t* pass_sorted = t.alloc<uint8_t>(px);
        auto* count = t.alloc<unsigned long long>(1);
        auto* prefix = t.alloc<unsigned long long>(20);
        k::roc_entries(d_est, d_gt, d_conf, n, theta, keys, pass, count, s);
        unsigned long long entries = 0;
        FMVS_CUDA_CHECK(cudaMemcpyAsync(&entries, count, sizeof(entries), cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
        if (entries == 0)
            fmvs::fail_input("roc: no valid estimates");  // evaluation.cpp:92-93
        k::RocSteps steps{};
        for (int step = 1; step <= 20; ++step) {  // evaluation.cpp:99-106
            const double density = step * 0.05;
            steps.m[step - 1] = static_cast<long long>(std::min<unsigned long long>(
                entries, static_cast<unsigned long long>(std::ceil(density * static_cast<double>(entries)))));
        }
        const size_t tb = k::roc_scratch_bytes(n);
        void* temp = t.alloc<uint8_t>(tb);
        k::roc_sort_prefix(keys, keys_sorted, pass, pass_sorted, n, temp, tb, steps, prefix, s);
        unsigned long long hp[20] = {};
        FMVS_CUDA_CHECK(cudaMemcpyAsync(hp, prefix, sizeof(hp), cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
        for (int step = 1; step <= 20; ++step) {
            const double density = step * 0.05;
            const unsigned long long m = static_cast<unsigned long long>(steps.m[step - 1]);
            densities[step - 1] = density;
            error_rates[step - 1] = 1.0 - static_cast<double>(hp[step - 1]) / m;
        }
    });
}

}  // extern "C"

// --------------------------------------- remaining reference helpers --
extern "C" {

int fmvs_gaussian_blur(fmvs_ctx* ctx, const uint8_t* image, int32_t w, int32_t h, int32_t radius,
                       double sigma, float* out) {
    return guarded([&] {
        ctx->use();
        if (radius < 0 || radius > 7)
            fmvs::fail_config("gaussian_blur: radius must be in 0..7");
        const size_t px = static_cast<size_t>(std::max(w, 0)) * std::max(h, 0);
        if (!px)
            return;
        const std::vector<double> kw = fmvs::blur_kernel(radius, sigma);
        k::BlurKernel bk{};
        bk.radius = radius;
        for (size_t i = 0; i < kw.size(); ++i)
            bk.w[i] = kw[i];
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const uint8_t* d_img = t.upload(image, px, s);
        float* tmp = t.alloc<float>(px);
        float* d_out = t.alloc<float>(px);
        k::gaussian_blur(d_img, w, h, bk, tmp, d_out, s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(out, d_out, px * 4, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int fmvs_census_transform(fmvs_ctx* ctx, const uint8_t* image, int32_t w, int32_t h, int32_t ww,
                          int32_t wh, uint64_t* out) {
    return guarded([&] {
        ctx->use();
        if (ww < 1 || wh < 1 || ww % 2 == 0 || wh % 2 == 0)  // matching.cpp:45-48
            fmvs::fail_config("census transform: window dimensions must be odd");
        if (ww * wh - 1 > 64)
            fmvs::fail_config("census transform: bit string exceeds 64 bits");
        const size_t px = static_cast<size_t>(std::max(w, 0)) * std::max(h, 0);
        if (!px)
            return;
        cudaStream_t s = ctx->stream;
        Tmp t(s);
        const uint8_t* d_img = t.upload(image, px, s);
        uint64_t* d_out = t.alloc<uint64_t>(px);
        k::census_transform(d_img, w, h, ww, wh, d_out, s);
        FMVS_CUDA_CHECK(cudaMemcpyAsync(out, d_out, px * 8, cudaMemcpyDeviceToHost, s));
        FMVS_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

uint64_t fmvs_census_bits_at(const uint8_t* image, int32_t w, int32_t h, int32_t x, int32_t y,
                             int32_t ww, int32_t wh) {
    const int rx = ww / 2, ry = wh / 2;  // matching.cpp:28-42
    const uint8_t c = image[static_cast<size_t>(y) * w + x];
    uint64_t bits = 0;
    for (int dy = -ry; dy <= ry; ++dy)
        for (int dx = -rx; dx <= rx; ++dx) {
            if (dx == 0 && dy == 0)
                continue;
            const int xx = std::min(std::max(x + dx, 0), w - 1), yy = std::min(std::max(y + dy, 0), h - 1);
            bits = (bits << 1) | (image[static_cast<size_t>(yy) * w + xx] < c ? 1u : 0u);
        }
    return bits;
}

int fmvs_ncc_cost(const float* a_in, const float* b_in, int32_t n, int32_t* cost) {
    return guarded([&] {
        if (n <= 0)  // matching.cpp:57-59
            fmvs::fail_input("ncc: patches must be non-empty and equal size");
        const double nn = static_cast<double>(n);
        double sa = 0, sb = 0, saa = 0, sbb = 0, sab = 0;
        for (int i = 0; i < n; ++i) {
            const double a = a_in[i], b = b_in[i];
            sa += a;
            sb += b;
            saa += a * a;
            sbb += b * b;
            sab += a * b;
        }
        const double var_a = saa - sa * sa / nn;
        const double var_b = sbb - sb * sb / nn;
        if (var_a <= 0.0 || var_b <= 0.0) {
            *cost = 255;
            return;
        }
        const double ncc = (sab - sa * sb / nn) / std::sqrt(var_a * var_b);
        const double c = 255.0 * std::min(1.0 - ncc, 1.0);
        *cost = static_cast<int32_t>(std::lround(std::clamp(c, 0.0, 255.0)));
    });
}

void fmvs_apply_homography(const double h[9], double x, double y, double out[2]) {
    // q = h * (x, y, 1), rows reduced left to right (the shim's order)
    const double qx = (h[0] * x + h[1] * y) + h[2] * 1.0;
    const double qy = (h[3] * x + h[4] * y) + h[5] * 1.0;
    const double qz = (h[6] * x + h[7] * y) + h[8] * 1.0;
    out[0] = qx / qz;
    out[1] = qy / qz;
}

int fmvs_cross_ratio(const double* p, int32_t dims, double* out) {
    return guarded([&] {
        if (dims != 2 && dims != 3)
            fmvs::fail_input("cross ratio: points must be 2D or 3D");
        auto dist = [&](int a, int b) {  // (p_b - p_a).norm()
            double acc = 0.0;
            for (int k2 = 0; k2 < dims; ++k2) {
                const double d = p[b * dims + k2] - p[a * dims + k2];
                acc = k2 == 0 ? d * d : acc + d * d;
            }
            return std::sqrt(acc);
        };
        const double d14 = dist(0, 3), d23 = dist(1, 2);  // geometry.cpp:159-165
        if (d14 == 0.0 || d23 == 0.0)
            fmvs::fail_input("cross ratio: coincident points p1=p4 or p2=p3");
        *out = dist(0, 2) * dist(1, 3) / (d14 * d23);
    });
}

int fmvs_require_centers_in_front(const double normal[3], double delta_min, const double* c, int32_t n) {
    return guarded([&] {
        for (int i = 0; i < n; ++i) {  // geometry.cpp:147-153
            const double d = (normal[0] * c[3 * i] + normal[1] * c[3 * i + 1]) + normal[2] * c[3 * i + 2];
            if (!(d + delta_min > 0.0))
                fmvs::fail_geometry("sweep geometry: camera center behind the near bounding plane");
        }
    });
}

}  // extern "C"
