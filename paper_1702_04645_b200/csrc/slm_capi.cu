// slm_capi.cu -- the extern "C" boundary (include/slm.h).  Every entry point catches
// SlmError / CUDA failures, records the message in the context and returns a code.
#include "slm_internal.cuh"
#include <cuda.h>
#include "../../include/slm.h"
#include <cstring>
#include <map>
#include <mutex>
#include <atomic>
#include <unordered_map>
#include <iterator>

double dbuf_now_ms() { return now_ms(); }

// ------------------------------------------------------------ device arena (DBuf)
// cudaMalloc / cudaFree cost milliseconds each at this footprint and vary run to run (a level
// loop makes hundreds of temporaries), so DBuf sub-allocates from one device arena reserved
// when the first context of the process is created: best-fit free blocks indexed by size,
// coalesced with their neighbours on release.  Requests the arena cannot hold fall back to
// cudaMalloc.  SLM_ARENA_GB sets the arena size (default 88% of the free device memory;
// 0 disables it).
namespace {
struct Arena {
    char *base = nullptr;
    size_t size = 0;
    std::map<size_t, size_t> by_off;              // free blocks: offset -> length
    std::multimap<size_t, size_t> by_len;         // free blocks: length -> offset
    std::unordered_map<void *, size_t> live;      // arena allocations: pointer -> length
};
constexpr size_t ARENA_ALIGN = 512;
constexpr int MAX_DEV = 64;
}
// heap objects never destroyed: static DBufs of other translation units release during exit
static std::mutex &g_dc_mu = *new std::mutex;
static Arena *g_arena = new Arena[MAX_DEV];

static void arena_insert_free(Arena &A, size_t off, size_t len) {
    auto nx = A.by_off.lower_bound(off);
    if (nx != A.by_off.end() && off + len == nx->first) {   // merge with the next block
        auto r = A.by_len.equal_range(nx->second);
        for (auto it = r.first; it != r.second; ++it)
            if (it->second == nx->first) { A.by_len.erase(it); break; }
        len += nx->second;
        nx = A.by_off.erase(nx);
    }
    if (nx != A.by_off.begin()) {                            // merge with the previous block
        auto pv = std::prev(nx);
        if (pv->first + pv->second == off) {
            auto r = A.by_len.equal_range(pv->second);
            for (auto it = r.first; it != r.second; ++it)
                if (it->second == pv->first) { A.by_len.erase(it); break; }
            off = pv->first;
            len += pv->second;
            A.by_off.erase(pv);
        }
    }
    A.by_off.emplace(off, len);
    A.by_len.emplace(len, off);
}

void dcache_reserve(int dev) {
    std::lock_guard<std::mutex> lk(g_dc_mu);
    Arena &A = g_arena[dev];
    if (A.base) return;
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    size_t want = (size_t)(0.88 * (double)fr);
    if (const char *e = getenv("SLM_ARENA_GB")) want = (size_t)(atof(e) * (double)(1ull << 30));
    want &= ~(size_t)(ARENA_ALIGN - 1);
    while (want >= (64ull << 20)) {
        void *p = nullptr;
        if (cudaMalloc(&p, want) == cudaSuccess) {
            A.base = (char *)p;
            A.size = want;
            A.by_off.emplace(0, want);
            A.by_len.emplace(want, 0);
            return;
        }
        cudaGetLastError();
        want /= 2;
    }
}

// the stream of the API call in progress on this thread (set by API_BEGIN)
static thread_local cudaStream_t g_tls_stream = nullptr;
static thread_local int g_tls_sms = 148;
int64_t slm_sms() { return g_tls_sms; }
struct PendingFree {
    int dev;
    size_t off, len;
    cudaEvent_t ev;
};
static std::vector<PendingFree> &g_pending = *new std::vector<PendingFree>;
static std::vector<cudaEvent_t> &g_event_pool = *new std::vector<cudaEvent_t>;
// blocks released while another context was alive become free once their stream passed
// the release point (called with g_dc_mu held)
static void drain_pending_locked() {
    for (size_t q = 0; q < g_pending.size();) {
        PendingFree &pf = g_pending[q];
        if (cudaEventQuery(pf.ev) == cudaSuccess) {
            arena_insert_free(g_arena[pf.dev], pf.off, pf.len);
            g_event_pool.push_back(pf.ev);
            pf = g_pending.back();
            g_pending.pop_back();
        } else {
            cudaGetLastError();
            q++;
        }
    }
}
void *dcache_alloc(size_t bytes, size_t *got) {
    const size_t need = (bytes + ARENA_ALIGN - 1) / ARENA_ALIGN * ARENA_ALIGN;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(g_dc_mu);
        if (!g_pending.empty()) drain_pending_locked();
        Arena &A = g_arena[dev];
        auto it = A.by_len.lower_bound(need);
        if (it != A.by_len.end()) {
            const size_t len = it->first, off = it->second;
            A.by_len.erase(it);
            A.by_off.erase(off);
            if (len > need) {
                A.by_off.emplace(off + need, len - need);
                A.by_len.emplace(len - need, off + need);
            }
            void *p = A.base + off;
            A.live.emplace(p, need);
            *got = need;
            return p;
        }
    }
    const double t = now_ms();
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, need);
    g_alloc_ms += now_ms() - t;
    g_alloc_calls++;
    if (getenv("SLM_ARENA_VERBOSE")) {
        std::lock_guard<std::mutex> lk(g_dc_mu);
        const Arena &A = g_arena[dev];
        const size_t largest = A.by_len.empty() ? 0 : A.by_len.rbegin()->first;
        size_t freeb = 0;
        for (auto &kv : A.by_off) freeb += kv.second;
        fprintf(stderr, "[arena] fallback cudaMalloc %.3f GB (arena %.1f GB, free %.2f GB, largest "
                "free %.2f GB) %.1f ms\n", need / 1e9, A.size / 1e9, freeb / 1e9, largest / 1e9,
                now_ms() - t);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        *got = 0;
        return nullptr;
    }
    *got = need;
    return p;
}
static std::atomic<int> g_live_ctx{0};

// DBuf registry: constructed on first use (file-scope static DBufs of other translation units
// are built during static initialisation) and never destroyed
struct DbufRegistry {
    std::mutex mu;
    std::unordered_map<void *, void (*)(void *)> live;
};
static DbufRegistry &dbuf_registry() {
    static DbufRegistry *r = new DbufRegistry;
    return *r;
}
void dbuf_track(void *self, void (*rel)(void *)) {
    DbufRegistry &R = dbuf_registry();
    std::lock_guard<std::mutex> lk(R.mu);
    R.live[self] = rel;
}
void dbuf_untrack(void *self) {
    DbufRegistry &R = dbuf_registry();
    std::lock_guard<std::mutex> lk(R.mu);
    R.live.erase(self);
}
void dbuf_release_all() {
    DbufRegistry &R = dbuf_registry();
    std::vector<std::pair<void *, void (*)(void *)>> all;
    {
        std::lock_guard<std::mutex> lk(R.mu);
        all.assign(R.live.begin(), R.live.end());
    }
    for (auto &kv : all) kv.second(kv.first);
}
void dcache_free(void *p, size_t bytes) {
    // Every kernel and copy of a context runs on its one stream, so a block released while
    // queued work still uses it is only handed to later work of the same stream (ordered
    // after it).  With several live contexts (several streams) the block is parked until an
    // event recorded on the releasing call's stream has completed.
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(g_dc_mu);
        Arena &A = g_arena[dev];
        auto it = A.live.find(p);
        if (it != A.live.end()) {
            const size_t len = it->second;
            const size_t off = (size_t)((char *)p - A.base);
            A.live.erase(it);
            if (g_live_ctx.load() > 1) {
                cudaEvent_t ev = nullptr;
                if (!g_event_pool.empty()) {
                    ev = g_event_pool.back();
                    g_event_pool.pop_back();
                } else if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
                    cudaGetLastError();
                    ev = nullptr;
                }
                if (ev && g_tls_stream && cudaEventRecord(ev, g_tls_stream) == cudaSuccess) {
                    g_pending.push_back({dev, off, len, ev});
                    return;
                }
                cudaGetLastError();
                if (ev) g_event_pool.push_back(ev);
                cudaDeviceSynchronize();   // no stream known: wait, as cudaFree did
            }
            arena_insert_free(A, off, len);
            return;
        }
    }
    (void)bytes;
    const double t = now_ms();
    cudaFree(p);
    g_alloc_ms += now_ms() - t;
    g_alloc_calls++;
}

void gen_rmat_device(slm_ctx *ctx, int scale, int edge_factor, double a, double b, double c,
                     uint64_t seed, int mode, DBuf<int32_t> &src, DBuf<int32_t> &dst,
                     DBuf<double> &w, int64_t &ne);
void gen_rgg_device(slm_ctx *ctx, int64_t n, double radius, uint64_t seed, DBuf<int32_t> &src,
                    DBuf<int32_t> &dst, DBuf<double> &w, int64_t &ne);

struct SlmStreamScope {   // the stream DBuf releases are ordered on during an API call,
    cudaStream_t prev;       // and the SM count grids are sized by
    int prev_sms;
    explicit SlmStreamScope(slm_ctx *c) : prev(g_tls_stream), prev_sms(g_tls_sms) {
        if (c) {
            g_tls_stream = c->stream;
            g_tls_sms = c->num_sms;
            cudaSetDevice(c->device);
        }
    }
    ~SlmStreamScope() {
        g_tls_stream = prev;
        g_tls_sms = prev_sms;
    }
};
#define API_BEGIN try { SlmStreamScope _slm_stream_scope(ctx);
#define API_END                                                                           \
    }                                                                                     \
    catch (const SlmError &e) {                                                           \
        if (ctx) ctx->err = e.msg;                                                        \
        return e.code;                                                                    \
    }                                                                                     \
    catch (const std::exception &e) {                                                     \
        if (ctx) ctx->err = e.what();                                                     \
        return SLM_ECUDA;                                                                 \
    }                                                                                     \
    return SLM_OK;

static void require_graph(slm_ctx *ctx) {
    SLM_REQUIRE(ctx->g != nullptr, SLM_ESTATE, "no graph loaded");
}
static void require_forest(slm_ctx *ctx) {
    require_graph(ctx);
    SLM_REQUIRE(ctx->f.n == ctx->g->n && ctx->f.a.p != nullptr && ctx->f.agg_valid &&
                    ctx->f.layout_valid,
                SLM_ESTATE, "no assignment forest for the current level");
}
static void require_agg(slm_ctx *ctx) {
    require_graph(ctx);
    SLM_REQUIRE(ctx->f.n == ctx->g->n && ctx->f.agg_valid, SLM_ESTATE,
                "no community labels for the current level");
}
static double gain_m(slm_ctx *ctx) { return ctx->g->m_w / ctx->gamma; }

__global__ void k_i64_to_i32(const int64_t *x, int64_t n, int32_t *y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = (int32_t)x[i];
}
// labels from the caller: range check against n, max, int32 copy
__global__ void k_labels_in(const int64_t *x, int64_t n, int32_t *y, int64_t *mx_bad) {
    long long mx = -1;
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = x[i];
        if (v < 0 || v >= n) {
            bad = 1;
            continue;
        }
        y[i] = (int32_t)v;
        mx = v > mx ? v : mx;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long om = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = om > mx ? om : mx;
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax((long long *)&mx_bad[0], mx);
        if (bad) atomicOr((unsigned long long *)&mx_bad[1], 1ull);
    }
}
__global__ void k_i32_to_i64b(const int32_t *x, int64_t n, int64_t *y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = x[i];
}

// host int64 -> device int32 (through a device staging buffer)
static void upload_i64_as_i32(slm_ctx *ctx, const int64_t *h, int64_t n, int32_t *d) {
    if (n == 0) return;
    int64_t *tmp = ctx->i64a.resize(n);
    CUDA_TRY(cudaMemcpyAsync(tmp, h, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    k_i64_to_i32<<<grid_for(n, 256), 256, 0, ctx->stream>>>(tmp, n, d);
}
static void download_i32_as_i64(slm_ctx *ctx, const int32_t *d, int64_t n, int64_t *h) {
    if (n == 0 || !h) return;
    int64_t *tmp = ctx->i64b.resize(n);
    k_i32_to_i64b<<<grid_for(n, 256), 256, 0, ctx->stream>>>(d, n, tmp);
    CUDA_TRY(cudaMemcpyAsync(h, tmp, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
}
static void download_i64(slm_ctx *ctx, const int64_t *d, int64_t n, int64_t *h) {
    if (n == 0 || !h) return;
    CUDA_TRY(cudaMemcpyAsync(h, d, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
}

static void new_level0(slm_ctx *ctx) {
    ctx->g0 = std::make_shared<LevelGraph>();
    ctx->g = ctx->g0;
    ctx->level = 0;
    ctx->f.n = -1;
    ctx->f.agg_valid = ctx->f.layout_valid = false;
    ctx->plan_version = ~0ull;
    ctx->wown_version = ~0ull;
}

extern "C" {

// Load every kernel of the library now instead of at its first launch (default lazy module
// loading: each first launch blocks the host for milliseconds).  Driver entry points: cuFuncGetModule,
// cuModuleGetFunctionCount, cuModuleEnumerateFunctions, cuFuncLoad (CUDA 12.4+); when any is
// unavailable the kernels simply keep loading lazily.
static void preload_modules() {
    typedef CUresult (*GetModule)(CUmodule *, CUfunction);
    typedef CUresult (*Count)(unsigned int *, CUmodule);
    typedef CUresult (*Enum)(CUfunction *, unsigned int, CUmodule);
    typedef CUresult (*Load)(CUfunction);
    void *p1 = nullptr, *p2 = nullptr, *p3 = nullptr, *p4 = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuFuncGetModule", &p1, cudaEnableDefault, &q) != cudaSuccess || !p1 ||
        cudaGetDriverEntryPoint("cuModuleGetFunctionCount", &p2, cudaEnableDefault, &q) != cudaSuccess || !p2 ||
        cudaGetDriverEntryPoint("cuModuleEnumerateFunctions", &p3, cudaEnableDefault, &q) != cudaSuccess || !p3 ||
        cudaGetDriverEntryPoint("cuFuncLoad", &p4, cudaEnableDefault, &q) != cudaSuccess || !p4) {
        cudaGetLastError();
        return;
    }
    const void *anchors[] = {slm_anchor_build(), slm_anchor_capi(), slm_anchor_commit(),
                             slm_anchor_forest(), slm_anchor_gen(), slm_anchor_level(),
                             slm_anchor_lgains(), slm_anchor_plan(), slm_anchor_positive(), slm_anchor_prim(), slm_anchor_surface(), slm_anchor_positive_lit(),
                             slm_anchor_sweep()};
    for (const void *a : anchors) {
        cudaFunction_t f;
        CUmodule mod;
        unsigned int cnt = 0;
        if (cudaGetFuncBySymbol(&f, a) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (((GetModule)p1)(&mod, (CUfunction)f) != CUDA_SUCCESS) continue;
        if (((Count)p2)(&cnt, mod) != CUDA_SUCCESS || cnt == 0) continue;
        std::vector<CUfunction> fs(cnt);
        if (((Enum)p3)(fs.data(), cnt, mod) != CUDA_SUCCESS) continue;
        for (CUfunction g : fs) ((Load)p4)(g);
    }
}

// context creation / destruction (and the release of the shared scratch with the last
// context) are serialised; a context itself is single-threaded (include/slm.h)
static std::mutex g_ctx_mu;

slm_ctx *slm_create(int device) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    slm_ctx *ctx = new slm_ctx();
    ctx->device = device;
    const char *pe = getenv("SLM_PROFILE");
    ctx->prof = pe && pe[0] == '1';
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        delete ctx;
        return nullptr;
    }
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (ctx->num_sms <= 0) ctx->num_sms = 148;
    // profiling runs synchronise at every phase boundary, so a lazy first-launch load would
    // be charged to the phase; preload there (and on request).  Otherwise the loads overlap
    // the asynchronously queued device work and preloading every kernel costs more (~0.2 s).
    g_live_ctx++;
    dcache_reserve(device);
    static bool preloaded = false;
    if (!preloaded && (ctx->prof || getenv("SLM_PRELOAD_MODULES"))) {
        preload_modules();
        preloaded = true;
    }
    return ctx;
}

void slm_destroy(slm_ctx *ctx) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    {
        SlmStreamScope scope(ctx);
        ctx->g.reset();
        ctx->g0.reset();
        ctx->scratch.clear();
    }
    cudaStreamSynchronize(ctx->stream2);
    cudaStreamDestroy(ctx->stream);
    cudaStreamDestroy(ctx->stream2);
    cudaEventDestroy(ctx->ev_fork);
    cudaEventDestroy(ctx->ev_join);
    delete ctx;
    // the last context: the static scratch kept across calls goes back to the arena too
    if (--g_live_ctx == 0) dbuf_release_all();
}

const char *slm_last_error(slm_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }
void *slm_stream(slm_ctx *ctx) { return ctx ? (void *)ctx->stream : nullptr; }

int slm_sync(slm_ctx *ctx) {
    API_BEGIN
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_build_graph(slm_ctx *ctx, int64_t n, const int64_t *src, const int64_t *dst,
                    const double *w, int64_t nedges) {
    API_BEGIN
    SLM_REQUIRE(n >= 0 && nedges >= 0, SLM_EINVAL, "negative size");
    for (int64_t e = 0; e < nedges; e++)
        SLM_REQUIRE(src[e] >= 0 && dst[e] >= 0 && src[e] < n && dst[e] < n, SLM_EINVAL,
                    "edge endpoint out of range");
    cudaSetDevice(ctx->device);
    new_level0(ctx);
    DBuf<int32_t> ds, dd;
    DBuf<double> dw;
    ds.resize(nedges);
    dd.resize(nedges);
    dw.resize(nedges);
    upload_i64_as_i32(ctx, src, nedges, ds.p);
    upload_i64_as_i32(ctx, dst, nedges, dd.p);
    if (nedges)
        CUDA_TRY(cudaMemcpyAsync(dw.p, w, nedges * 8, cudaMemcpyHostToDevice, ctx->stream));
    build_level_from_edges(ctx, *ctx->g, n, ds.p, dd.p, dw.p, nedges);
    API_END
}

int slm_build_graph_device(slm_ctx *ctx, int64_t n, const int32_t *d_src, const int32_t *d_dst,
                           const double *d_w, int64_t nedges) {
    API_BEGIN
    cudaSetDevice(ctx->device);
    new_level0(ctx);
    build_level_from_edges(ctx, *ctx->g, n, d_src, d_dst, d_w, nedges);
    API_END
}

int slm_build_rmat(slm_ctx *ctx, int scale, int edge_factor, double a, double b, double c,
                   uint64_t seed, int weight_mode) {
    API_BEGIN
    cudaSetDevice(ctx->device);
    new_level0(ctx);
    DBuf<int32_t> s, d;
    DBuf<double> w;
    int64_t ne = 0;
    gen_rmat_device(ctx, scale, edge_factor, a, b, c, seed, weight_mode, s, d, w, ne);
    build_level_from_edges(ctx, *ctx->g, int64_t(1) << scale, s.p, d.p, w.p, ne);
    API_END
}

int slm_build_rgg(slm_ctx *ctx, int64_t n, double radius, uint64_t seed) {
    API_BEGIN
    cudaSetDevice(ctx->device);
    new_level0(ctx);
    DBuf<int32_t> s, d;
    DBuf<double> w;
    int64_t ne = 0;
    gen_rgg_device(ctx, n, radius, seed, s, d, w, ne);
    build_level_from_edges(ctx, *ctx->g, n, s.p, d.p, w.p, ne);
    API_END
}

int slm_build_pairs(slm_ctx *ctx, int32_t mode, int64_t n, int64_t blocks, double p_in,
                    double p_out, const int32_t *comm, const double *kin, const double *kout,
                    const double *K, int64_t n_comms, double O, uint64_t seed) {
    API_BEGIN
    SLM_REQUIRE(n >= 0 && n < (int64_t(1) << 31) && (mode == 0 || mode == 1), SLM_EINVAL,
                "bad pair-model arguments");
    SLM_REQUIRE(mode == 0 || (comm && kin && kout && K && n_comms > 0), SLM_EINVAL,
                "DC-SBM needs comm, kin, kout, K");
    cudaSetDevice(ctx->device);
    new_level0(ctx);
    DBuf<int32_t> dc;
    DBuf<double> dki, dko, dK;
    if (mode == 1) {
        dc.resize(n);
        dki.resize(n);
        dko.resize(n);
        dK.resize(n_comms);
        CUDA_TRY(cudaMemcpyAsync(dc.p, comm, n * 4, cudaMemcpyHostToDevice, ctx->stream));
        CUDA_TRY(cudaMemcpyAsync(dki.p, kin, n * 8, cudaMemcpyHostToDevice, ctx->stream));
        CUDA_TRY(cudaMemcpyAsync(dko.p, kout, n * 8, cudaMemcpyHostToDevice, ctx->stream));
        CUDA_TRY(cudaMemcpyAsync(dK.p, K, n_comms * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    const PairArgs P = make_pair_args(mode, n, blocks, p_in, p_out, dc.p, dki.p, dko.p, dK.p, O, seed);
    DBuf<int32_t> src, dst;
    DBuf<double> w;
    int64_t ne = 0;
    gen_pairs_device(ctx, P, src, dst, w, ne);
    build_level_from_edges(ctx, *ctx->g, n, src.p, dst.p, w.p, ne);
    API_END
}

int slm_graph_info(slm_ctx *ctx, int64_t *n, int64_t *ne, int64_t *ue, double *m_w,
                   int32_t *flags) {
    API_BEGIN
    require_graph(ctx);
    const LevelGraph &G = *ctx->g;
    if (n) *n = G.n;
    if (ne) *ne = G.ne;
    if (ue) *ue = G.ue;
    if (m_w) *m_w = G.m_w;
    if (flags) {
        // plan-sweep path of this level (run_plan): 4 = exact uint32 group sums (integer
        // weights, every row total < 2^32), else fp64 on integer sums (exact), else the
        // sorted reference-order form (real-valued weights)
        const bool sorted = getenv("SLM_PLAN_SORTED") != nullptr;
        const bool u32 = G.u32_ok && !getenv("SLM_FORCE_GENERIC") && !sorted;
        *flags = (G.sym ? 1 : 0) | (G.integral ? 2 : 0) | (u32 ? 4 : 0) | (sorted ? 8 : 0);
    }
    API_END
}

int slm_get_csr(slm_ctx *ctx, int64_t *out_ptr, int64_t *out_dst, double *out_w) {
    API_BEGIN
    require_graph(ctx);
    const LevelGraph &G = *ctx->g;
    download_i64(ctx, G.csr_ptr.p, G.n + 1, out_ptr);
    download_i32_as_i64(ctx, G.csr_dst.p, G.ne, out_dst);
    if (out_w && G.ne)
        CUDA_TRY(cudaMemcpyAsync(out_w, G.csr_w.p, G.ne * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_get_union(slm_ctx *ctx, int64_t *ptr, int64_t *nbr, double *u) {
    API_BEGIN
    require_graph(ctx);
    const LevelGraph &G = *ctx->g;
    download_i64(ctx, G.uptr.p, G.n + 1, ptr);
    download_i32_as_i64(ctx, G.unbr.p, G.ue, nbr);
    if (u && G.ue)
        CUDA_TRY(cudaMemcpyAsync(u, G.uu.p, G.ue * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_get_union_rows(slm_ctx *ctx, int64_t r0, int64_t r1, int64_t *ptr_out, int64_t *nbr_out,
                       double *u_out) {
    API_BEGIN
    require_graph(ctx);
    const LevelGraph &G = *ctx->g;
    SLM_REQUIRE(r0 >= 0 && r0 <= r1 && r1 <= G.n, SLM_EINVAL, "row range out of bounds");
    std::vector<int64_t> p(r1 - r0 + 1);
    CUDA_TRY(cudaMemcpy(p.data(), G.uptr.p + r0, (r1 - r0 + 1) * 8, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i <= r1 - r0; i++) ptr_out[i] = p[i] - p[0];
    const int64_t cnt = p[r1 - r0] - p[0];
    if (nbr_out && cnt) {
        std::vector<int32_t> tmp(cnt);
        CUDA_TRY(cudaMemcpy(tmp.data(), G.unbr.p + p[0], cnt * 4, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < cnt; i++) nbr_out[i] = tmp[i];
    }
    if (u_out && cnt)
        CUDA_TRY(cudaMemcpy(u_out, G.uu.p + p[0], cnt * 8, cudaMemcpyDeviceToHost));
    API_END
}

int slm_get_csr_rows(slm_ctx *ctx, int64_t r0, int64_t r1, int64_t *ptr_out, int64_t *dst_out,
                     double *w_out) {
    API_BEGIN
    require_graph(ctx);
    const LevelGraph &G = *ctx->g;
    SLM_REQUIRE(r0 >= 0 && r0 <= r1 && r1 <= G.n, SLM_EINVAL, "row range out of bounds");
    std::vector<int64_t> p(r1 - r0 + 1);
    CUDA_TRY(cudaMemcpy(p.data(), G.csr_ptr.p + r0, (r1 - r0 + 1) * 8, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i <= r1 - r0; i++) ptr_out[i] = p[i] - p[0];
    const int64_t cnt = p[r1 - r0] - p[0];
    if (dst_out && cnt) {
        std::vector<int32_t> tmp(cnt);
        CUDA_TRY(cudaMemcpy(tmp.data(), G.csr_dst.p + p[0], cnt * 4, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < cnt; i++) dst_out[i] = tmp[i];
    }
    if (w_out && cnt)
        CUDA_TRY(cudaMemcpy(w_out, G.csr_w.p + p[0], cnt * 8, cudaMemcpyDeviceToHost));
    API_END
}

int slm_get_strengths(slm_ctx *ctx, double *s_out, double *s_in) {
    API_BEGIN
    require_graph(ctx);
    const LevelGraph &G = *ctx->g;
    if (G.n) {
        if (s_out)
            CUDA_TRY(cudaMemcpyAsync(s_out, G.s_out.p, G.n * 8, cudaMemcpyDeviceToHost, ctx->stream));
        if (s_in)
            CUDA_TRY(cudaMemcpyAsync(s_in, G.s_in.p, G.n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_set_resolution(slm_ctx *ctx, double gamma) {
    API_BEGIN
    SLM_REQUIRE(gamma > 0.0 && std::isfinite(gamma), SLM_EINVAL, "resolution must be > 0");
    ctx->gamma = gamma;
    ctx->plan_version = ~0ull;
    ctx->wown_version = ~0ull;
    API_END
}

int slm_assign(slm_ctx *ctx, int64_t *a_out) {
    API_BEGIN
    require_graph(ctx);
    const LevelGraph &G = *ctx->g;
    Forest &F = ctx->f;
    F.a.resize(G.n);
    F.n = G.n;
    F.agg_valid = F.layout_valid = false;
    run_assign(ctx, G, gain_m(ctx), F.a.p);
    download_i32_as_i64(ctx, F.a.p, G.n, a_out);
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_set_assignment(slm_ctx *ctx, const int64_t *a) {
    API_BEGIN
    require_graph(ctx);
    const LevelGraph &G = *ctx->g;
    for (int64_t i = 0; i < G.n; i++)
        SLM_REQUIRE(a[i] >= 0 && a[i] < G.n, SLM_EINVAL, "assignment out of range");
    Forest &F = ctx->f;
    F.a.resize(G.n);
    F.n = G.n;
    upload_i64_as_i32(ctx, a, G.n, F.a.p);
    forest_refresh(ctx, G, F);
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

static void copy_forest_out(slm_ctx *ctx, int64_t *a_out, int64_t *comm_out, uint8_t *oc_out,
                            int64_t *n_comms) {
    Forest &F = ctx->f;
    download_i32_as_i64(ctx, F.a.p, F.n, a_out);
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    download_i32_as_i64(ctx, F.comm.p, F.n, comm_out);
    if (oc_out && F.n)
        CUDA_TRY(cudaMemcpyAsync(oc_out, F.on_cycle.p, F.n, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (n_comms) *n_comms = F.n_comms;
}

int slm_components(slm_ctx *ctx, int64_t *comm_out, uint8_t *on_cycle_out, int64_t *n_comms) {
    API_BEGIN
    require_graph(ctx);
    Forest &F = ctx->f;
    SLM_REQUIRE(F.n == ctx->g->n && F.a.p, SLM_ESTATE, "no assignment");
    forest_refresh(ctx, *ctx->g, F);
    copy_forest_out(ctx, nullptr, comm_out, on_cycle_out, n_comms);
    API_END
}

int slm_get_forest(slm_ctx *ctx, int64_t *a_out, int64_t *comm_out, uint8_t *on_cycle_out,
                   int64_t *n_comms) {
    API_BEGIN
    require_forest(ctx);
    copy_forest_out(ctx, a_out, comm_out, on_cycle_out, n_comms);
    API_END
}

int slm_get_aggregates(slm_ctx *ctx, double *S_out, double *S_in, int64_t *count) {
    API_BEGIN
    require_agg(ctx);
    Forest &F = ctx->f;
    int64_t nc = F.n_comms;
    if (S_out) CUDA_TRY(cudaMemcpyAsync(S_out, F.S_out.p, nc * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (S_in) CUDA_TRY(cudaMemcpyAsync(S_in, F.S_in.p, nc * 8, cudaMemcpyDeviceToHost, ctx->stream));
    download_i32_as_i64(ctx, F.count.p, nc, count);
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_local_gains(slm_ctx *ctx, double *lg_out) {
    API_BEGIN
    require_agg(ctx);
    const LevelGraph &G = *ctx->g;
    DBuf<double> lg;
    DBuf<uint8_t> bad;
    lg.resize(G.n);
    bad.resize(ctx->f.n_comms);
    run_local_gains(ctx, G, ctx->f, gain_m(ctx), lg.p, bad.p);
    if (lg_out && G.n)
        CUDA_TRY(cudaMemcpyAsync(lg_out, lg.p, G.n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_positive(slm_ctx *ctx, const slm_config *cfg, int64_t *splits, int64_t *unresolved,
                 int32_t *changed, double *gains_out, int64_t gains_cap) {
    API_BEGIN
    require_forest(ctx);
    const LevelGraph &G = *ctx->g;
    std::vector<double> gains;
    int ch = 0;
    int64_t sp = 0, un = 0;
    run_positive(ctx, G, ctx->f, gain_m(ctx), cfg ? cfg->scc_cut_cap : 10000, &sp, &un, &ch,
                 gains_out ? &gains : nullptr);
    if (ch) forest_refresh(ctx, G, ctx->f);
    if (splits) *splits = sp;
    if (unresolved) *unresolved = un;
    if (changed) *changed = ch;
    if (gains_out)
        for (int64_t k = 0; k < (int64_t)gains.size() && k < gains_cap; k++) gains_out[k] = gains[k];
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_plan_sweep(slm_ctx *ctx, const int64_t *comm_in, int64_t *cstar_out) {
    API_BEGIN
    require_graph(ctx);
    const LevelGraph &G = *ctx->g;
    Forest &F = ctx->f;
    if (comm_in) {
        // explicit snapshot: labels + aggregates from them (members/aggregates only);
        // range check and max label on the device
        F.n = G.n;
        F.comm.resize(G.n);
        int64_t *tmp = ctx->i64a.resize(G.n > 0 ? G.n : 1);
        if (G.n)
            CUDA_TRY(cudaMemcpyAsync(tmp, comm_in, G.n * 8, cudaMemcpyHostToDevice, ctx->stream));
        int64_t *dmx = ctx->i64b.resize(2);
        const int64_t init[2] = {-1, 0};
        CUDA_TRY(cudaMemcpyAsync(dmx, init, 16, cudaMemcpyHostToDevice, ctx->stream));
        k_labels_in<<<grid_for(G.n, 256), 256, 0, ctx->stream>>>(tmp, G.n, F.comm.p, dmx);
        int64_t hmx[2];
        CUDA_TRY(cudaMemcpyAsync(hmx, dmx, 16, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        SLM_REQUIRE(hmx[1] == 0, SLM_EINVAL, "labels out of range");
        F.n_comms = hmx[0] + 1;
        build_members_and_aggregates(ctx, G, F);
        F.layout_valid = false;
        F.version++;
    } else {
        require_forest(ctx);
    }
    ctx->cstar.resize(G.n);
    run_plan(ctx, G, F, gain_m(ctx), ctx->cstar.p);
    download_i32_as_i64(ctx, ctx->cstar.p, G.n, cstar_out);
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_plan_sweep_async(slm_ctx *ctx, int32_t bin_mask) {
    API_BEGIN
    require_agg(ctx);
    const LevelGraph &G = *ctx->g;
    ctx->cstar.resize(G.n);
    run_plan(ctx, G, ctx->f, gain_m(ctx), ctx->cstar.p, bin_mask, nullptr);
    API_END
}

int slm_plan_groups(slm_ctx *ctx, int64_t *groups, int64_t *bin_rows, int64_t *bin_entries) {
    API_BEGIN
    require_agg(ctx);
    const LevelGraph &G = *ctx->g;
    DBuf<unsigned long long> d;
    d.resize(1);
    CUDA_TRY(cudaMemsetAsync(d.p, 0, 8, ctx->stream));
    ctx->cstar.resize(G.n);
    run_plan(ctx, G, ctx->f, gain_m(ctx), ctx->cstar.p, 127, d.p);
    unsigned long long h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, d.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (groups) *groups = (int64_t)h;
    if (bin_rows)
        for (int b = 0; b < NBINS; b++) bin_rows[b] = G.bin_off[b + 1] - G.bin_off[b];
    if (bin_entries)
        for (int b = 0; b < NBINS; b++) bin_entries[b] = G.bin_entries[b];
    API_END
}

int slm_debug_sweep_floor(slm_ctx *ctx, int32_t mode, double *ms) {
    API_BEGIN
    require_agg(ctx);
    SLM_REQUIRE(ctx->g->u32_ok, SLM_EUNSUP, "needs the integer fast path");
    *ms = sweep_floor_ms(ctx, *ctx->g, ctx->f, mode);
    API_END
}

int slm_debug_sort(slm_ctx *ctx, int32_t kind, void *keys, void *vals, int64_t n, int32_t end_bit,
                   double *ms) {
    API_BEGIN
    SLM_REQUIRE(ctx && keys && vals && n >= 0 && (kind == 0 || kind == 1), SLM_EINVAL,
                "bad sort arguments");
    SLM_REQUIRE(end_bit >= 0 && end_bit <= (kind == 0 ? 64 : 32), SLM_EINVAL, "bad end_bit");
    const double t = n ? debug_sort(ctx, kind, keys, vals, n, end_bit) : 0.0;
    if (ms) *ms = t;
    API_END
}

int slm_debug_scan(slm_ctx *ctx, int32_t kind, const void *in, void *out, const uint32_t *keys,
                   int64_t n) {
    API_BEGIN
    SLM_REQUIRE(ctx && in && out && n >= 0 && kind >= 0 && kind <= 4 && (kind != 4 || keys),
                SLM_EINVAL, "bad scan arguments");
    if (n) debug_scan(ctx, kind, in, out, keys, n);
    API_END
}

// ---------------------------------------------------------- the level loop in one call
// run() of detector.py:548-653 without a host round trip per phase: ASSIGN, COMPONENTS,
// POSITIVE, {MAXIMAL -> POSITIVE} up to max_outer_iters, AGGREGATE, until the identity
// level.  Same stop rules, statistics and exact fast-forward as paper_1702_04645_b200/
// detector.py (which calls this when no per-phase trace or debug check is requested).
// stats[0..4]: accepted_moves, accepted_splits, unresolved_negative, skipped POSITIVE
// calls, levels that hit max_outer_iters; phase_s[0..4]: assign, components, positive,
// maximal, aggregate (host wall seconds, the reference's tick()).
int slm_run(slm_ctx *ctx, const slm_config *cfg, int64_t *n_levels, int64_t *stats,
            double *phase_s) {
    API_BEGIN
    require_graph(ctx);
    SLM_REQUIRE(cfg && cfg->max_outer_iters >= 1, SLM_EINVAL, "bad config");
    SLM_REQUIRE(ctx->g->n > 0, SLM_EINVAL, "graph has no nodes");
    ctx->run_levels.clear();
    ctx->run_sweeps.clear();
    ctx->run_paths.clear();
    int64_t st[5] = {0, 0, 0, 0, 0};
    double ph[5] = {0, 0, 0, 0, 0};
    auto clk = [] { return now_ms() * 1e-3; };
    auto ok = [&](int rc) {
        if (rc != SLM_OK) throw SlmError{rc, ctx->err};
    };
    int64_t level = 0;
    for (;;) {
        const LevelGraph &G = *ctx->g;
        const int64_t n_level = G.n;
        const bool integral = G.integral;
        int32_t fl = 0;
        ok(slm_graph_info(ctx, nullptr, nullptr, nullptr, nullptr, &fl));
        ctx->run_paths.push_back(fl & 4 ? 0 : ((fl & 2) && !(fl & 8) ? 1 : 2));
        double t = clk();
        ok(slm_assign(ctx, nullptr));
        ph[0] += clk() - t;
        t = clk();
        int64_t nc = 0;
        ok(slm_components(ctx, nullptr, nullptr, &nc));
        ph[1] += clk() - t;
        t = clk();
        int64_t sp = 0, un = 0;
        int32_t ch = 0;
        ok(slm_positive(ctx, cfg, &sp, &un, &ch, nullptr, 0));
        ph[2] += clk() - t;
        st[1] += sp;
        st[2] += un;
        int64_t last_un = un;
        int64_t sweeps = 0;
        for (;;) {
            if (sweeps >= cfg->max_outer_iters) {
                st[4]++;
                ctx->run_paths.back() |= 8;   // stopped by the cap (the reference warns)
                break;
            }
            t = clk();
            int32_t imp = 0;
            int64_t app = 0;
            ok(slm_maximal(ctx, cfg, level, sweeps, &imp, &app, nullptr, 0));
            ph[3] += clk() - t;
            sweeps++;
            st[0] += app;
            if (!imp) break;
            if (app == 0 && integral) {   // forest unchanged: POSITIVE would repeat itself
                st[2] += last_un;
                st[3]++;
                continue;
            }
            t = clk();
            ok(slm_positive(ctx, cfg, &sp, &un, &ch, nullptr, 0));
            ph[2] += clk() - t;
            st[1] += sp;
            st[2] += un;
            last_un = un;
        }
        ctx->run_sweeps.push_back(sweeps);
        std::vector<int64_t> lab(n_level);
        ok(slm_get_forest(ctx, nullptr, lab.data(), nullptr, &nc));
        ctx->run_levels.push_back(std::move(lab));
        if (nc == n_level) break;
        t = clk();
        ok(slm_aggregate(ctx));
        ph[4] += clk() - t;
        level++;
    }
    *n_levels = (int64_t)ctx->run_levels.size();
    if (stats)
        for (int k = 0; k < 5; k++) stats[k] = st[k];
    if (phase_s)
        for (int k = 0; k < 5; k++) phase_s[k] = ph[k];
    API_END
}

int slm_run_level(slm_ctx *ctx, int64_t t, int64_t *n_nodes, int64_t *sweeps, int32_t *plan_path,
                  int64_t *labels_out) {
    API_BEGIN
    SLM_REQUIRE(t >= 0 && t < (int64_t)ctx->run_levels.size(), SLM_EINVAL, "no such level");
    const std::vector<int64_t> &L = ctx->run_levels[t];
    if (n_nodes) *n_nodes = (int64_t)L.size();
    if (sweeps) *sweeps = ctx->run_sweeps[t];
    if (plan_path) *plan_path = (int32_t)ctx->run_paths[t];
    if (labels_out) std::copy(L.begin(), L.end(), labels_out);
    API_END
}

// ----------------------------------------------------- reference API surface helpers

int slm_community_sums(slm_ctx *ctx, int64_t n, const int64_t *labels, int64_t n_comms,
                       const double *s_out, const double *s_in, double *S_out, double *S_in,
                       int64_t *count) {
    API_BEGIN
    SLM_REQUIRE(n >= 0 && n_comms >= 0 && n_comms < (int64_t(1) << 31), SLM_EINVAL, "bad sizes");
    for (int64_t i = 0; i < n; i++)
        SLM_REQUIRE(labels[i] >= 0 && labels[i] < n_comms, SLM_EINVAL, "label out of range");
    cudaStream_t s = ctx->stream;
    DBuf<int32_t> lab, cnt;
    DBuf<double> so, si, So, Si;
    lab.resize(n); so.resize(n); si.resize(n);
    cnt.resize(n_comms); So.resize(n_comms); Si.resize(n_comms);
    upload_i64_as_i32(ctx, labels, n, lab.p);
    if (n) {
        CUDA_TRY(cudaMemcpyAsync(so.p, s_out, n * 8, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(si.p, s_in, n * 8, cudaMemcpyHostToDevice, s));
    }
    comm_sums_device(ctx, lab.p, n, n_comms, so.p, si.p, So.p, Si.p, cnt.p);
    std::vector<int32_t> c(n_comms);
    if (n_comms) {
        CUDA_TRY(cudaMemcpyAsync(S_out, So.p, n_comms * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(S_in, Si.p, n_comms * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(c.data(), cnt.p, n_comms * 4, cudaMemcpyDeviceToHost, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int64_t k = 0; k < n_comms; k++) count[k] = c[k];
    API_END
}

int slm_gain_switch(slm_ctx *ctx, const int64_t *labels, const int64_t *nodes, int64_t k,
                    int64_t frm, int64_t to, const double *agg4, double m, double *gain) {
    API_BEGIN
    require_graph(ctx);
    const LevelGraph &G = *ctx->g;
    SLM_REQUIRE(k >= 0, SLM_EINVAL, "negative node count");
    for (int64_t q = 0; q < k; q++)
        SLM_REQUIRE(nodes[q] >= 0 && nodes[q] < G.n, SLM_EINVAL, "node out of range");
    if (to >= 0 && to == frm) {
        *gain = 0.0;
    } else {
        DBuf<int32_t> lab, nd;
        lab.resize(G.n);
        nd.resize(k);
        upload_i64_as_i32(ctx, labels, G.n, lab.p);
        upload_i64_as_i32(ctx, nodes, k, nd.p);
        *gain = gain_switch_device(ctx, G, lab.p, nd.p, k, (int32_t)frm, (int32_t)(to < 0 ? -1 : to),
                                   agg4, m);
    }
    API_END
}

int slm_reverse_assignment(slm_ctx *ctx, int64_t n, const int64_t *a, int64_t *ptr_out,
                           int64_t *kids_out, int64_t *n_kids) {
    API_BEGIN
    SLM_REQUIRE(n >= 0 && n < (int64_t(1) << 31), SLM_EINVAL, "bad size");
    for (int64_t i = 0; i < n; i++)
        SLM_REQUIRE(a[i] >= 0 && a[i] < n, SLM_EINVAL, "assignment out of range");
    DBuf<int32_t> da;
    da.resize(n);
    upload_i64_as_i32(ctx, a, n, da.p);
    reverse_assignment_device(ctx, da.p, n, ptr_out, kids_out, n_kids);
    API_END
}

int slm_get_union_split(slm_ctx *ctx, double *w_out, double *w_in) {
    API_BEGIN
    require_graph(ctx);
    const LevelGraph &G = *ctx->g;
    DBuf<double> wo, wi;
    wo.resize(G.ue);
    wi.resize(G.ue);
    union_split_device(ctx, G, wo.p, wi.p);
    if (G.ue) {
        CUDA_TRY(cudaMemcpyAsync(w_out, wo.p, G.ue * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_TRY(cudaMemcpyAsync(w_in, wi.p, G.ue * 8, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_canonicalize_labels(slm_ctx *ctx, int64_t n, const int64_t *labels, int64_t *out,
                            int64_t *n_comms) {
    API_BEGIN
    SLM_REQUIRE(n >= 0 && n < (int64_t(1) << 31), SLM_EINVAL, "bad size");
    int64_t lo = 0, hi = -1;
    for (int64_t i = 0; i < n; i++) {
        if (i == 0 || labels[i] < lo) lo = labels[i];
        if (i == 0 || labels[i] > hi) hi = labels[i];
    }
    SLM_REQUIRE(n == 0 || (uint64_t)(hi - lo) < (uint64_t(1) << 32) - 1, SLM_EINVAL,
                "label range exceeds 2^32");
    std::vector<uint32_t> off(n);
    for (int64_t i = 0; i < n; i++) off[i] = (uint32_t)(labels[i] - lo);
    DBuf<uint32_t> dl;
    DBuf<int32_t> dout;
    dl.resize(n);
    dout.resize(n);
    if (n) CUDA_TRY(cudaMemcpyAsync(dl.p, off.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
    *n_comms = canonicalize_device(ctx, dl.p, n, bits_for(hi - lo + 2), dout.p);
    download_i32_as_i64(ctx, dout.p, n, out);
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_build_aggregate(slm_ctx *ctx, slm_ctx *src, const int64_t *labels, int64_t n_comms) {
    API_BEGIN
    SLM_REQUIRE(src && src->g, SLM_ESTATE, "source context has no graph");
    SLM_REQUIRE(src->device == ctx->device, SLM_EINVAL, "contexts on different devices");
    const LevelGraph &G = *src->g;
    SLM_REQUIRE(n_comms >= 0 && n_comms <= G.n, SLM_EINVAL, "bad community count");
    for (int64_t i = 0; i < G.n; i++)
        SLM_REQUIRE(labels[i] >= 0 && labels[i] < n_comms, SLM_EINVAL, "label out of range");
    CUDA_TRY(cudaStreamSynchronize(src->stream));
    DBuf<int32_t> lab;
    lab.resize(G.n);
    upload_i64_as_i32(ctx, labels, G.n, lab.p);
    auto next = std::make_shared<LevelGraph>();
    run_aggregate(ctx, G, lab.p, n_comms, *next);
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    new_level0(ctx);
    ctx->g0 = next;
    ctx->g = next;
    API_END
}

int slm_get_cstar(slm_ctx *ctx, int64_t *cstar_out) {
    API_BEGIN
    require_graph(ctx);
    SLM_REQUIRE(ctx->cstar.n == (size_t)ctx->g->n, SLM_ESTATE, "no plan computed");
    download_i32_as_i64(ctx, ctx->cstar.p, ctx->g->n, cstar_out);
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_maximal(slm_ctx *ctx, const slm_config *cfg, int64_t level, int64_t sweep,
                int32_t *improved, int64_t *applied, double *gains_out, int64_t gains_cap) {
    API_BEGIN
    require_forest(ctx);
    SLM_REQUIRE(cfg && cfg->accept_prob > 0.0 && cfg->accept_prob <= 1.0, SLM_EINVAL,
                "accept_prob must be in (0, 1]");
    const LevelGraph &G = *ctx->g;
    Forest &F = ctx->f;
    const double m = gain_m(ctx);
    // the plan depends only on the forest: reuse it across coin-only sweeps (F7)
    if (ctx->plan_version != F.version || ctx->cstar.n != (size_t)G.n) {
        ctx->cstar.resize(G.n);
        phase_mark(ctx, -1);
        ctx->wown_version = ~0ull;
        ctx->wown_fresh = false;
        run_plan(ctx, G, F, m, ctx->cstar.p);
        phase_mark(ctx, PH_PLAN);
        ctx->plan_version = F.version;
        if (ctx->wown_fresh) ctx->wown_version = F.version;   // the view sweep wrote it
    }
    int imp = 0;
    int64_t app = 0;
    std::vector<double> gains;
    const bool keep_wown = ctx->wown_version == F.version && G.u32_ok;
    run_commit(ctx, G, F, m, ctx->cstar.p, cfg->seed, cfg->accept_prob, level, sweep, &imp, &app,
               gains_out ? &gains : nullptr, keep_wown ? ctx->wown.p : nullptr);
    if (app) {
        forest_refresh(ctx, G, F);
        // the commit carried wown over to the new partition (same components, new ids)
        ctx->wown_version = keep_wown ? F.version : ~0ull;
    }
    if (improved) *improved = imp;
    if (applied) *applied = app;
    if (gains_out)
        for (int64_t k = 0; k < (int64_t)gains.size() && k < gains_cap; k++) gains_out[k] = gains[k];
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_aggregate(slm_ctx *ctx) {
    API_BEGIN
    require_forest(ctx);
    auto next = std::make_shared<LevelGraph>();
    run_aggregate(ctx, *ctx->g, ctx->f.comm.p, ctx->f.n_comms, *next);
    ctx->g = next;
    ctx->level++;
    ctx->f.n = -1;
    ctx->f.agg_valid = ctx->f.layout_valid = false;
    ctx->plan_version = ~0ull;
    ctx->wown_version = ~0ull;
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_score(slm_ctx *ctx, int32_t on_original, const int64_t *labels, double gamma,
              double *q_out) {
    API_BEGIN
    require_graph(ctx);
    const LevelGraph &G = on_original ? *ctx->g0 : *ctx->g;
    DBuf<int32_t> lab;
    lab.resize(G.n);
    for (int64_t i = 0; i < G.n; i++)
        SLM_REQUIRE(labels[i] >= 0 && labels[i] < (int64_t(1) << 31), SLM_EINVAL, "bad label");
    upload_i64_as_i32(ctx, labels, G.n, lab.p);
    *q_out = run_score(ctx, G, lab.p, gamma);
    API_END
}

__global__ void k_uniform(uint64_t base, const int64_t *ids, int64_t k, double *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = uniform01_at(base, ids[i]);
}

int slm_uniform01(slm_ctx *ctx, uint64_t seed, int64_t level, int64_t sweep, const int64_t *ids,
                  int64_t k, double *out) {
    API_BEGIN
    if (k == 0) return SLM_OK;
    DBuf<int64_t> d;
    DBuf<double> o;
    d.resize(k);
    o.resize(k);
    CUDA_TRY(cudaMemcpyAsync(d.p, ids, k * 8, cudaMemcpyHostToDevice, ctx->stream));
    k_uniform<<<grid_for(k, 256), 256, 0, ctx->stream>>>(mix_key2(seed, level, sweep), d.p, k, o.p);
    CUDA_TRY(cudaMemcpyAsync(out, o.p, k * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    API_END
}

int slm_phase_times(slm_ctx *ctx, double *ms, int32_t nmax, int32_t reset) {
    API_BEGIN
    for (int i = 0; i < NPHASE && i < nmax; i++) ms[i] = ctx->ph_ms[i];
    // two extra slots: host ms spent in cudaMalloc / cudaFree and the number of such calls
    // (process-wide)
    if (nmax > NPHASE) ms[NPHASE] = g_alloc_ms;
    if (nmax > NPHASE + 1) ms[NPHASE + 1] = (double)g_alloc_calls;
    // ... and the host ms spent building sweep views (always measured; once per level)
    if (nmax > NPHASE + 2) ms[NPHASE + 2] = ctx->view_build_ms;
    if (reset) {
        ctx->view_build_ms = 0.0;
        for (int i = 0; i < NPHASE; i++) ctx->ph_ms[i] = 0.0;
        g_alloc_ms = 0.0;
        g_alloc_calls = 0;
    }
    API_END
}

int slm_last_commit_stats(slm_ctx *ctx, int64_t *candidates, int64_t *rounds) {
    API_BEGIN
    if (candidates) *candidates = ctx->last_candidates;
    if (rounds) *rounds = ctx->last_rounds;
    API_END
}

}  // extern "C"

// a kernel of this translation unit (module preloading, slm_capi.cu preload_modules)
const void *slm_anchor_capi() { return (const void *)k_i64_to_i32; }
