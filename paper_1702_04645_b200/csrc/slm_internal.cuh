// slm_internal.cuh -- shared device/host plumbing of the sm_100a SLM library.
//
// Compiled with -fmad=false: every fp64 gain expression below is evaluated with the
// reference's operand order and IEEE rounding of each + - * /, never contracted to FMA,
// so integer-weighted graphs (all sums exact below 2^53) reproduce the reference bit for
// bit.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>
#include <unordered_map>
#include <memory>
#include <memory>

#define SLM_OK 0
#define SLM_EINVAL (-1)
#define SLM_ECUDA (-2)
#define SLM_ENOMEM (-3)
#define SLM_ESTATE (-4)
#define SLM_EUNSUP (-5)

struct SlmError {
    int code;
    std::string msg;
};

#define CUDA_TRY(expr)                                                                   \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess)                                                           \
            throw SlmError{_e == cudaErrorMemoryAllocation ? SLM_ENOMEM : SLM_ECUDA,     \
                           std::string(#expr) + ": " + cudaGetErrorString(_e)};          \
    } while (0)

#define SLM_REQUIRE(cond, code, msg)                                                     \
    do {                                                                                 \
        if (!(cond)) throw SlmError{(code), (msg)};                                      \
    } while (0)

// ------------------------------------------------------------------ device buffers

// host time spent in device allocation calls and their number (diagnostics, phase_times)
inline double g_alloc_ms = 0.0;
inline long long g_alloc_calls = 0;
double dbuf_now_ms();

// Device memory behind DBuf: a per-device arena reserved at context creation, sub-allocated
// best-fit with coalescing (slm_capi.cu); cudaMalloc only beyond it.
void *dcache_alloc(size_t bytes, size_t *got);
void dcache_free(void *p, size_t bytes);
void dcache_reserve(int device);
// every live DBuf is tracked, so the grow-only scratch kept in static DBufs across calls can be
// returned to the arena when the last context goes away (slm_destroy)
void dbuf_track(void *self, void (*rel)(void *));
void dbuf_untrack(void *self);
void dbuf_release_all();

template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;     // logical length
    size_t cap = 0;   // allocated elements
    DBuf() { dbuf_track(this, [](void *self) { static_cast<DBuf *>(self)->release(); }); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    ~DBuf() {
        release();
        dbuf_untrack(this);
    }
    void release() {
        if (p) dcache_free(p, cap * sizeof(T));
        p = nullptr;
        n = cap = 0;
    }
    // grow-only; contents are not preserved when reallocating
    T *resize(size_t cnt) {
        if (cnt > cap) {
            release();
            size_t c = cnt ? cnt : 1;
            size_t got = 0;
            p = (T *)dcache_alloc(c * sizeof(T), &got);
            if (!p) CUDA_TRY(cudaErrorMemoryAllocation);
            cap = got / sizeof(T);
        }
        n = cnt;
        return p;
    }
    void swap(DBuf &o) {
        std::swap(p, o.p);
        std::swap(n, o.n);
        std::swap(cap, o.cap);
    }
    size_t bytes() const { return n * sizeof(T); }
};

// --------------------------------------------------------------- level graph state

// union rows are binned by degree d; bin b holds BIN_LO[b] <= d <= BIN_HI[b]
constexpr int NBINS = 6;
__host__ __device__ constexpr int64_t bin_hi(int b) {
    return b == 0 ? 32 : b == 1 ? 256 : b == 2 ? 1024 : b == 3 ? 4096 : b == 4 ? 16383 : INT64_MAX;
}
constexpr int SMALL_MAX = 32;     // warp lanes = entries (packed rows)
constexpr int TINY_MAX = 8;       // bin-0 rows up to this degree: one lane per row
constexpr int HALF_MAX = 64;      // bin-1 rows up to this degree: one half-warp per row
constexpr int MID_MAX = 4096;     // generic path: CTA-per-row shared-memory hash up to here

constexpr int HUB_SEG = 4096;     // entries per hub-row work item of the integer sweep
constexpr int64_t HUB_BIG_DEG = 32768;   // hub rows spread over CTAs by segment above this

struct SweepView;
struct slm_ctx;
struct Forest;

// Canonical directed CSR + neighbour union + strengths of one hierarchy level
// (graph.py:63-175, 257-263).  Node ids int32, entry offsets int64.
struct LevelGraph {
    int64_t n = 0, ne = 0, ue = 0;
    DBuf<int64_t> csr_ptr;
    DBuf<int32_t> csr_dst;
    DBuf<double> csr_w;
    DBuf<int64_t> uptr;
    DBuf<int32_t> unbr;
    DBuf<double> uu;          // w_out + w_in (F6)
    DBuf<uint32_t> uu32;      // compact u when integral and every row total < 2^32
    bool u32_ok = false;
    DBuf<double> s_out, s_in;
    DBuf<double2> s2;         // {s_out, s_in} interleaved (one sector per node)
    double m_w = 0.0;
    bool sym = false;         // W == W^T (then s_in == s_out bitwise)
    bool integral = false;    // all weights integer-valued, m_w < 2^53
    // degree bins of union rows (ascending row ids inside each bin)
    DBuf<int32_t> bin_rows;
    int64_t bin_off[NBINS + 1] = {0, 0, 0, 0, 0, 0, 0};
    int64_t bin_entries[NBINS] = {0, 0, 0, 0, 0, 0};
    int64_t bin0_tiny = 0;     // bin-0 rows: the first bin0_tiny have d <= TINY_MAX (stable partition)
    int64_t bin1_half = 0;     // sweep view only: the last bin1_half bin-1 rows have d <= HALF_MAX
    DBuf<int64_t> large_hoff;  // per row with d > MID_MAX (bins 4, 5): global hash offset
    int64_t large_hash_total = 0;
    // bin-5 (hub) rows of the integer sweep, in processing order j (descending degree):
    // work items (j << 20 | segment); bin-5 row index, table offset and size of row j
    DBuf<int64_t> hub_seg, hub_row, hub_off, hub_size;
    mutable DBuf<uint32_t> hub_gprev;   // per hub row: groups found by the previous sweep (0: unknown)
    int64_t hub_nseg = 0, hub_rows_n = 0, hub_ring = 0;   // hub_ring: arena slots
    int64_t hub_big_rows = 0, hub_big_items = 0;        // rows with d > HUB_BIG_DEG (prefix)
    int32_t max_deg = 0;
    // degree-ordered copy of the union for the integer plan sweep (built on first use)
    mutable std::shared_ptr<SweepView> view;
    // nodes whose union rows exceed the POSITIVE warp executor's budget (found on first use)
    mutable DBuf<int32_t> heavy_nodes;
    mutable int64_t heavy_n = 0;
    mutable bool heavy_valid = false;
};

// The integer plan sweep's view of a level: union rows renumbered by descending degree
// (stable by id), neighbour ids mapped to the new numbering.  Group sums are exact integers
// and the argmax compares community ids, so the sweep over the view yields the reference's
// targets bit for bit; the numbering only changes where labels and rows sit in memory
// (hub rows and the labels of hub neighbours become contiguous and cache-resident).
struct SweepView {
    LevelGraph V;                 // n, ue, uptr, unbr (view ids), uu32, s_out / s2, bins, hubs
    DBuf<int32_t> order;          // view row k -> node
    DBuf<int32_t> vlabel, vcstar; // per sweep: labels and targets in view order
    DBuf<uint32_t> vwown;         // per sweep: own-community group sums in view order
};
SweepView &ensure_sweep_view(slm_ctx *ctx, const LevelGraph &G);
void view_gather_labels(slm_ctx *ctx, SweepView &W, const int32_t *label);   // vlabel = label[order]
void wown_to_node_order(slm_ctx *ctx, const LevelGraph &G);   // scatter vwown -> ctx->wown if pending
void run_local_gains_wown(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m,
                          const uint32_t *wown, double *d_lg, uint8_t *d_bad);
void commit_wown_deltas(slm_ctx *ctx, const LevelGraph &G, const int32_t *pre, const int32_t *post,
                        uint32_t *wown);
void build_bins(slm_ctx *ctx, LevelGraph &G);

// Assignment forest + derived community structure (forest.py:23-67, quality.py:52-79).
struct Forest {
    int64_t n = 0, n_comms = 0;
    DBuf<int32_t> a, comm;
    DBuf<uint8_t> on_cycle;
    DBuf<int32_t> cptr, members;        // members sorted by (comm, node)
    DBuf<int32_t> croot;                // per community: smallest cycle node (DFS root)
    DBuf<double> S_out, S_in;
    DBuf<double2> S2;                   // {S_out, S_in} interleaved
    DBuf<float> S1f;                    // float(S_out) (approximate pass of the sweep)
    DBuf<float2> S2f;                   // float {S_out, S_in}
    DBuf<int32_t> count;
    // DFS pre-order layout per community (root = smallest cycle node)
    DBuf<int32_t> order, pos, sz, kptr, kids;
    bool layout_valid = false;
    bool agg_valid = false;
    uint64_t version = 0;
};

enum Phase { PH_PLAN, PH_CAND, PH_SPEC, PH_WALK, PH_REFRESH_COMP, PH_REFRESH_AGG, PH_REFRESH_LAYOUT,
             PH_POS_LG, PH_POS_SMALL, PH_POS_GIANT, PH_ASSIGN, PH_AGGREGATE, NPHASE };

struct slm_ctx {
    // optional phase timing (SLM_PROFILE=1): synchronises at phase boundaries
    bool prof = false;
    double ph_ms[NPHASE] = {};
    double ph_t0 = 0.0;
    int device = 0;
    int num_sms = 148;           // cudaDevAttrMultiProcessorCount of the device
    // per-context (= per-device) "function attributes set" flags: the opt-in dynamic shared
    // memory size of a kernel is a per-device property
    bool sweep_attr_set[2] = {false, false};
    bool giant_attr_set = false;
    double view_build_ms = 0.0;  // host ms spent building sweep views (once per level)
    int walk_blocks = 0;         // co-resident grid of the persistent commit walker (cached)
    cudaStream_t stream = nullptr;
    cudaStream_t stream2 = nullptr;              // side stream of the plan sweep (hub rows)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::string err;
    std::shared_ptr<LevelGraph> g0, g;   // original graph and current level
    Forest f;
    double gamma = 1.0;
    int64_t level = 0;
    // plan cache (exact fast-forward of coin-only sweeps)
    DBuf<int32_t> cstar;
    uint64_t plan_version = ~0ull;
    // own-community group sum per node (integer sweep by-product, node order) and the forest
    // version it is exact for: POSITIVE's local gains reuse it, kept exact across a commit by
    // deltas over the moved nodes' rows (~0: invalid)
    DBuf<uint32_t> wown;
    uint64_t wown_version = ~0ull;
    bool wown_fresh = false;   // set by the view sweep that just wrote wown
    bool wown_in_view = false; // wown still in the sweep view's row order (vwown), not scattered
    // scratch
    DBuf<uint8_t> tmp;           // scan / sort status and histogram scratch (slm_prim.cu)
    DBuf<uint64_t> sort_k64;     // radix sort ping-pong buffers
    DBuf<double> sort_v64;
    DBuf<uint32_t> sort_k32;
    DBuf<int32_t> sort_v32;
    DBuf<int64_t> i64a, i64b;
    DBuf<int32_t> i32a, i32b, i32c, i32d;
    DBuf<double> f64a, f64b;
    DBuf<uint64_t> u64a, u64b;
    DBuf<double> hash_vals;
    DBuf<int32_t> hash_keys;
    DBuf<int2> hub_tab;          // hub tables {community, sum} of the integer sweep (kept empty)
    DBuf<uint32_t> hub_occ;      // occupied-slot lists (same offsets)
    DBuf<uint32_t> hub_cnt;      // per hub row: list length (kept zero between sweeps)
    DBuf<uint32_t> hub_ovf;      // per hub row: overflow flag; fallback row list; its count
    DBuf<int32_t> ovf_rows;      // rows of bins 2-4 whose communities overflowed the shared table
    DBuf<uint32_t> ovf_cnt;      // [0] overflow rows, [1 + b] list length of overflow CTA b
    DBuf<int2> ovf_tab;          // per overflow CTA: global table (kept empty)
    DBuf<uint32_t> ovf_occ;
    // sweep-view build scratch (grow-only, reused by every level)
    DBuf<uint32_t> view_k0, view_k1;
    DBuf<int32_t> view_i0, view_nid;
    DBuf<int64_t> view_deg, view_bound;
    int32_t *h_flag = nullptr;   // pinned host scalars
    int64_t *h_i64 = nullptr;
    double *h_f64 = nullptr;
    // counters of the last phase calls
    int64_t last_rounds = 0, last_candidates = 0, last_accepted = 0;
    int64_t last_pos_warnings = 0;   // scc_cut_cap peels of the last POSITIVE call
    // results of the last slm_run (labels per level on the host, per-level sweeps / paths)
    std::vector<std::vector<int64_t>> run_levels;
    std::vector<int64_t> run_sweeps, run_paths;
    // per-context grow-only scratch of the phase functions (CTX_SCRATCH below)
    std::unordered_map<const void *, std::shared_ptr<void>> scratch;
};

// Grow-only scratch kept across calls, owned by the context (released with it): the
// phase functions' scratch is per context, so several contexts (threads, devices) never
// share device buffers.
template <class T>
T &ctx_scratch(slm_ctx *ctx, const void *tag) {
    std::shared_ptr<void> &p = ctx->scratch[tag];
    if (!p) p = std::shared_ptr<void>(new T(), [](void *q) { delete static_cast<T *>(q); });
    return *static_cast<T *>(p.get());
}
#define CTX_SCRATCH(T, name)                                                               \
    static const char name##_tag_ = 0;                                                     \
    T &name = ctx_scratch<T>(ctx, &name##_tag_)

// ------------------------------------------------------------------------- helpers

#include <chrono>
static inline double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
}
// mark the end of a phase (no-op unless profiling)
static inline void phase_mark(slm_ctx *ctx, int ph) {
    if (!ctx->prof) return;
    cudaStreamSynchronize(ctx->stream);
    double t = now_ms();
    if (ph >= 0) ctx->ph_ms[ph] += t - ctx->ph_t0;
    ctx->ph_t0 = t;
}

// SM count of the device of the API call in flight (set with the call's stream, slm_capi.cu)
int64_t slm_sms();
#define SMS() slm_sms()

static inline unsigned grid_for(int64_t work, int block, int64_t cap = SMS() * 64) {
    int64_t g = (work + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// numpy DOUBLE_pairwise_sum, device twin of oracle/slm_oracle.c pw_sum (used where a
// single thread owns a short segment).
__host__ __device__ inline double pw_leaf(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; i++) r += a[i];
        return r;
    }
    double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8) {
        r0 += a[i + 0]; r1 += a[i + 1]; r2 += a[i + 2]; r3 += a[i + 3];
        r4 += a[i + 4]; r5 += a[i + 5]; r6 += a[i + 6]; r7 += a[i + 7];
    }
    double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    for (; i < n; i++) res += a[i];
    return res;
}

// iterative pairwise (explicit stack) for one thread: exact numpy order for any n
__host__ __device__ inline double pw_sum_seq(const double *a, int64_t n) {
    if (n <= 128) return pw_leaf(a, n);
    // emulate recursion: stack of (offset, len, state); results combined left+right
    struct Fr { int64_t off, len; double left; int st; };
    Fr stk[48];
    double ret = 0.0;
    int sp = 0;
    stk[0] = {0, n, 0.0, 0};
    while (sp >= 0) {
        Fr &fr = stk[sp];
        if (fr.len <= 128) {
            ret = pw_leaf(a + fr.off, fr.len);
            sp--;
            continue;
        }
        int64_t n2 = fr.len / 2;
        n2 -= n2 % 8;
        if (fr.st == 0) {
            fr.st = 1;
            stk[sp + 1] = {fr.off, n2, 0.0, 0};
            sp++;
        } else if (fr.st == 1) {
            fr.left = ret;
            fr.st = 2;
            stk[sp + 1] = {fr.off + n2, fr.len - n2, 0.0, 0};
            sp++;
        } else {
            ret = fr.left + ret;
            sp--;
        }
    }
    return ret;
}

// np.add.reduceat segment: first + pairwise(rest)
__host__ __device__ inline double reduceat_seq(const double *a, int64_t n) {
    return a[0] + pw_sum_seq(a + 1, n - 1);
}

// ---------------------------------------------------------------- counter RNG

#define RNG_GAMMA 0x9E3779B97F4A7C15ULL
#define RNG_MIX1 0xBF58476D1CE4E5B9ULL
#define RNG_MIX2 0x94D049BB133111EBULL

__host__ __device__ inline uint64_t fin64(uint64_t z) {   // rng.py:19-23
    z = (z ^ (z >> 30)) * RNG_MIX1;
    z = (z ^ (z >> 27)) * RNG_MIX2;
    return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t mix_key2(uint64_t seed, int64_t level, int64_t sweep) {
    uint64_t s = fin64(seed);                                  // rng.py:26-31
    s = fin64(s + RNG_GAMMA + (uint64_t)level);
    s = fin64(s + RNG_GAMMA + (uint64_t)sweep);
    return s;
}
__host__ __device__ inline double uniform01_at(uint64_t base, int64_t id) {   // rng.py:34-43
    uint64_t z = fin64((uint64_t)id * RNG_GAMMA + base);
    return (double)(z >> 11) * 0x1.0p-53;
}

// ------------------------------------------------------------- internal API

void build_level_from_edges(slm_ctx *ctx, LevelGraph &G, int64_t n, const int32_t *d_src,
                            const int32_t *d_dst, const double *d_w, int64_t ne_in);
void build_level_from_keys(slm_ctx *ctx, LevelGraph &G, int64_t n, DBuf<uint64_t> &keys,
                           DBuf<double> &vals, int64_t ne_in);
double device_pairwise_sum(slm_ctx *ctx, const double *d_a, int64_t n);
void run_assign(slm_ctx *ctx, const LevelGraph &G, double m, int32_t *d_a);
void run_components(slm_ctx *ctx, Forest &F, int64_t n);
void build_members_and_aggregates(slm_ctx *ctx, const LevelGraph &G, Forest &F);
void build_layout(slm_ctx *ctx, Forest &F);
void run_plan(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m, int32_t *d_cstar,
              int bin_mask = 127, unsigned long long *d_groups = nullptr);
double sweep_floor_ms(slm_ctx *ctx, const LevelGraph &G, Forest &F, int mode);
void run_plan_u32(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m, int32_t *d_cstar,
                  int bin_mask, unsigned long long *d_groups);
void run_local_gains(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m, double *d_lg,
                     uint8_t *d_bad);
void run_positive(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m, int64_t scc_cap,
                  int64_t *splits, int64_t *unresolved, int *changed, std::vector<double> *gains);
void run_commit(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m, const int32_t *d_cstar,
                uint64_t seed, double accept_prob, int64_t level, int64_t sweep, int *improved,
                int64_t *applied, std::vector<double> *gains, uint32_t *wown = nullptr);
void run_aggregate(slm_ctx *ctx, const LevelGraph &G, const int32_t *d_labels, int64_t n_comms,
                   LevelGraph &out);
double run_score(slm_ctx *ctx, const LevelGraph &G, const int32_t *d_labels, double gamma);
void forest_refresh(slm_ctx *ctx, const LevelGraph &G, Forest &F);   // comps + agg + layout

// slm_gen.cu: pair-model generators (SBM / DC-SBM), one Bernoulli draw per node pair
struct PairArgs {
    int mode;
    int64_t n, bs;
    double p_in, p_out, O;
    const int32_t *comm;
    const double *kin, *kout, *K;
    uint64_t base;
};
PairArgs make_pair_args(int mode, int64_t n, int64_t blocks, double p_in, double p_out,
                        const int32_t *d_comm, const double *d_kin, const double *d_kout,
                        const double *d_K, double O, uint64_t seed);
void gen_pairs_device(slm_ctx *ctx, const PairArgs &P, DBuf<int32_t> &src, DBuf<int32_t> &dst,
                      DBuf<double> &w, int64_t &ne);

// slm_prim.cu: single-pass decoupled look-back scans and the onesweep LSD radix sort
template <class TI, class TO>
void dev_exclusive_sum(slm_ctx *ctx, const TI *in, TO *out, int64_t n);
void dev_exclusive_sum_by_key(slm_ctx *ctx, const uint32_t *keys, const int32_t *in, int32_t *out,
                              int64_t n);
void sort_pairs_u64_f64(slm_ctx *ctx, DBuf<uint64_t> &keys, DBuf<double> &vals, int64_t n,
                        int end_bit);
void sort_pairs_u32_i32(slm_ctx *ctx, uint32_t *keys_in, uint32_t *keys_out, int32_t *vals_in,
                        int32_t *vals_out, int64_t n, int end_bit);
bool sort_pairs_u32_u64(slm_ctx *ctx, uint32_t *kA, uint32_t *kB, uint64_t *vA, uint64_t *vB,
                        int64_t n, int end_bit);
int bits_for(int64_t v);
double debug_sort(slm_ctx *ctx, int kind, void *keys, void *vals, int64_t n, int end_bit);
void debug_scan(slm_ctx *ctx, int kind, const void *in, void *out, const uint32_t *keys, int64_t n);

// one kernel per translation unit: their modules are loaded at context creation
const void *slm_anchor_build();
const void *slm_anchor_capi();
const void *slm_anchor_commit();
const void *slm_anchor_forest();
const void *slm_anchor_gen();
const void *slm_anchor_level();
const void *slm_anchor_lgains();
const void *slm_anchor_plan();
const void *slm_anchor_positive();
const void *slm_anchor_prim();
const void *slm_anchor_surface();
const void *slm_anchor_positive_lit();
void bad_cycle_lengths(slm_ctx *ctx, const Forest &F, const int32_t *d_list, int32_t nbad,
                       std::vector<int32_t> &h_len);
void run_positive_literal(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m,
                          int64_t scc_cap, const std::vector<int2> &ranges,
                          std::vector<std::vector<double>> &gains, std::vector<int32_t> &unres,
                          std::vector<int32_t> &changed, int64_t *nwarn);

// slm_surface.cu: the rest of the reference's hot-path API surface
void comm_sums_device(slm_ctx *ctx, const int32_t *d_lab, int64_t n, int64_t nc,
                      const double *d_so, const double *d_si, double *d_So, double *d_Si,
                      int32_t *d_cnt);
double gain_switch_device(slm_ctx *ctx, const LevelGraph &G, const int32_t *d_lab,
                          const int32_t *d_nodes, int64_t k, int32_t frm, int32_t to,
                          const double agg[4], double m);
void reverse_assignment_device(slm_ctx *ctx, const int32_t *d_a, int64_t n, int64_t *h_ptr,
                               int64_t *h_kids, int64_t *h_nk);
void union_split_device(slm_ctx *ctx, const LevelGraph &G, double *d_wo, double *d_wi);
int64_t canonicalize_device(slm_ctx *ctx, const uint32_t *d_lab, int64_t n, int end_bit,
                            int32_t *d_out);
const void *slm_anchor_sweep();
