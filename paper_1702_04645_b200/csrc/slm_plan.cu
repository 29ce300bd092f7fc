// slm_plan.cu -- the O(E) sweeps over the neighbour union.
//
//   ASSIGN  (_assign_targets, detector.py:123-146): per row the first neighbour maximising
//           g = (u/m) - ((s_out[r]*s_in[j] + s_in[r]*s_out[j])/m2); self unless max > 0.
//   PLAN    (_best_targets, detector.py:367-418, the local-move sweep): per row, sum u per
//           neighbouring community, t_c = (gsum/m) - ((s_out*S_in' + s_in*S_out')/m2) with
//           the node's own strengths removed from its own community, then the lowest c != L
//           attaining max t_c, taken only if it strictly beats staying.
//   LOCAL GAINS (local_gains, quality.py:170-183): weight to own community -> gain; flags
//           the communities POSITIVE must examine (detector.py:341-345).
//
// Degree-binned: rows with <= 32 union entries run one warp per row with lanes = entries
// and __match_any_sync grouping by community; rows up to 4096 entries run one CTA per row
// with an open-addressing hash in shared memory; hub rows run one CTA per row over a hash
// table in global scratch.  Group sums use atomics only where all summands are integers
// (then any order is exact); the argmax is a lexicographic (t desc, c asc) reduction, so
// results never depend on scheduling.
#include "slm_internal.cuh"

struct PlanArgs {
    const int64_t *uptr;
    const int32_t *unbr;
    const double *uu;
    const int32_t *label;
    const double *S_out, *S_in;
    const double *s_out, *s_in;
    double m, m2;
    int32_t *cstar;
    unsigned long long *groups;   // distinct (node, community) groups seen (roofline G)
};

__device__ __forceinline__ bool better(double t1, int32_t c1, double t2, int32_t c2) {
    return t1 > t2 || (t1 == t2 && c1 < c2);
}

__device__ __forceinline__ void warp_argmax(double &t, int32_t &c) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        double ot = __shfl_xor_sync(0xffffffffu, t, off);
        int32_t oc = __shfl_xor_sync(0xffffffffu, c, off);
        if (better(ot, oc, t, c)) {
            t = ot;
            c = oc;
        }
    }
}

// t_c of _best_targets (detector.py:400-402)
__device__ __forceinline__ double plan_gain(double gsum, bool own, double so, double si,
                                            double Sin_c, double Sout_c, double m, double m2) {
    double sin_c = Sin_c - (own ? si : 0.0);
    double sout_c = Sout_c - (own ? so : 0.0);
    return gsum / m - (so * sin_c + si * sout_c) / m2;
}

// ------------------------------------------------------------------ PLAN small

__global__ void __launch_bounds__(256) k_plan_small(PlanArgs A, const int32_t *rows, int64_t nrows) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (; w < nrows; w += nw) {
        const int32_t r = rows[w];
        const int64_t e0 = A.uptr[r];
        const int d = (int)(A.uptr[r + 1] - e0);
        const int32_t L = A.label[r];
        const double so = A.s_out[r], si = A.s_in[r];
        const bool valid = lane < d;
        int32_t c = -1;
        double wt = 0.0;
        if (valid) {
            c = A.label[A.unbr[e0 + lane]];
            wt = A.uu[e0 + lane];
        }
        const unsigned mask = __match_any_sync(0xffffffffu, c);
        double gs = 0.0;
        for (int k = 0; k < d; k++) {
            double v = __shfl_sync(0xffffffffu, wt, k);
            if ((mask >> k) & 1u) gs += v;
        }
        const bool leader = valid && (lane == __ffs(mask) - 1);
        const bool own = (c == L);
        if (A.groups) {
            unsigned lm = __ballot_sync(0xffffffffu, leader);
            if (lane == 0) atomicAdd(A.groups, (unsigned long long)__popc(lm));
        }
        double t = -INFINITY;
        if (leader) t = plan_gain(gs, own, so, si, A.S_in[c], A.S_out[c], A.m, A.m2);
        const unsigned ownmask = __ballot_sync(0xffffffffu, leader && own);
        double t_own = __shfl_sync(0xffffffffu, t, ownmask ? (__ffs(ownmask) - 1) : 0);
        double bt = (leader && !own) ? t : -INFINITY;
        int32_t bc = (leader && !own) ? c : 0x7fffffff;
        warp_argmax(bt, bc);
        if (lane == 0) {
            double t_stay = ownmask ? t_own
                                    : -(so * (A.S_in[L] - si) + si * (A.S_out[L] - so)) / A.m2;
            A.cstar[r] = (bc != 0x7fffffff && bt > t_stay) ? bc : L;
        }
    }
}

// ------------------------------------------------------- PLAN mid / large (hash)

__device__ __forceinline__ uint32_t hslot(int32_t c, uint32_t hmask) {
    return ((uint32_t)c * 2654435761u) & hmask;
}

template <int BLOCK>
__device__ void block_argmax(double &t, int32_t &c, double *sh_t, int32_t *sh_c) {
    warp_argmax(t, c);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sh_t[wid] = t;
        sh_c[wid] = c;
    }
    __syncthreads();
    if (wid == 0) {
        t = lane < BLOCK / 32 ? sh_t[lane] : -INFINITY;
        c = lane < BLOCK / 32 ? sh_c[lane] : 0x7fffffff;
        warp_argmax(t, c);
    }
    __syncthreads();
}

// one CTA per row; hk/hv either shared (mid) or global scratch (large)
template <int BLOCK>
__device__ void plan_row_hash(const PlanArgs &A, int32_t r, int32_t *hk, double *hv, uint32_t H,
                              double *sh_t, int32_t *sh_c, double *sh_stay) {
    const int64_t e0 = A.uptr[r], e1 = A.uptr[r + 1];
    const int32_t L = A.label[r];
    const double so = A.s_out[r], si = A.s_in[r];
    const uint32_t hmask = H - 1;
    for (uint32_t k = threadIdx.x; k < H; k += BLOCK) {
        hk[k] = -1;
        hv[k] = 0.0;
    }
    if (threadIdx.x == 0) *sh_stay = NAN;
    __syncthreads();
    for (int64_t e = e0 + threadIdx.x; e < e1; e += BLOCK) {
        int32_t c = A.label[A.unbr[e]];
        double wt = A.uu[e];
        uint32_t sl = hslot(c, hmask);
        for (;;) {
            int32_t prev = atomicCAS(&hk[sl], -1, c);
            if (prev == -1 || prev == c) {
                atomicAdd(&hv[sl], wt);
                break;
            }
            sl = (sl + 1) & hmask;
        }
    }
    __syncthreads();
    double bt = -INFINITY;
    int32_t bc = 0x7fffffff;
    unsigned ng = 0;
    for (uint32_t k = threadIdx.x; k < H; k += BLOCK) {
        int32_t c = hk[k];
        if (c < 0) continue;
        ng++;
        bool own = (c == L);
        double t = plan_gain(hv[k], own, so, si, A.S_in[c], A.S_out[c], A.m, A.m2);
        if (own) *sh_stay = t;
        else if (better(t, c, bt, bc)) {
            bt = t;
            bc = c;
        }
    }
    if (A.groups) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) ng += __shfl_xor_sync(0xffffffffu, ng, off);
        if ((threadIdx.x & 31) == 0 && ng) atomicAdd(A.groups, (unsigned long long)ng);
    }
    __syncthreads();
    block_argmax<BLOCK>(bt, bc, sh_t, sh_c);
    if (threadIdx.x == 0) {
        double t_stay = *sh_stay;
        if (t_stay != t_stay)   // no neighbour in own community
            t_stay = -(so * (A.S_in[L] - si) + si * (A.S_out[L] - so)) / A.m2;
        A.cstar[r] = (bc != 0x7fffffff && bt > t_stay) ? bc : L;
    }
    __syncthreads();
}

constexpr int MID_BLOCK = 256;
constexpr int MID_H = 2 * MID_MAX;   // 8192 slots: 32 KB keys + 64 KB sums

__global__ void __launch_bounds__(MID_BLOCK) k_plan_mid(PlanArgs A, const int32_t *rows, int64_t nrows) {
    extern __shared__ __align__(16) unsigned char smem[];
    double *hv = (double *)smem;
    int32_t *hk = (int32_t *)(smem + MID_H * sizeof(double));
    __shared__ double sh_t[MID_BLOCK / 32];
    __shared__ int32_t sh_c[MID_BLOCK / 32];
    __shared__ double sh_stay;
    for (int64_t i = blockIdx.x; i < nrows; i += gridDim.x) {
        int32_t r = rows[i];
        int64_t d = A.uptr[r + 1] - A.uptr[r];
        uint32_t H = 64;
        while (H < 2 * d) H <<= 1;
        plan_row_hash<MID_BLOCK>(A, r, hk, hv, H, sh_t, sh_c, &sh_stay);
    }
}

constexpr int LARGE_BLOCK = 1024;
__global__ void __launch_bounds__(LARGE_BLOCK) k_plan_large(PlanArgs A, const int32_t *rows,
                                                          int64_t nrows, const int64_t *hoff,
                                                          int32_t *gk, double *gv) {
    __shared__ double sh_t[LARGE_BLOCK / 32];
    __shared__ int32_t sh_c[LARGE_BLOCK / 32];
    __shared__ double sh_stay;
    for (int64_t i = blockIdx.x; i < nrows; i += gridDim.x) {
        int32_t r = rows[i];
        uint32_t H = (uint32_t)(hoff[i + 1] - hoff[i]);
        plan_row_hash<LARGE_BLOCK>(A, r, gk + hoff[i], gv + hoff[i], H, sh_t, sh_c, &sh_stay);
    }
}

static PlanArgs make_args(const LevelGraph &G, const Forest &F, double m, int32_t *cstar) {
    PlanArgs A;
    A.groups = nullptr;
    A.uptr = G.uptr.p;
    A.unbr = G.unbr.p;
    A.uu = G.uu.p;
    A.label = F.comm.p;
    A.S_out = F.S_out.p;
    A.S_in = F.S_in.p;
    A.s_out = G.s_out.p;
    A.s_in = G.s_in.p;
    A.m = m;
    A.m2 = m * m;
    A.cstar = cstar;
    return A;
}

__global__ void k_copy_labels(const int32_t *label, int64_t n, int32_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = label[i];
}

// --------------------------------------------- PLAN, sorted form (real-valued weights)
// The reference's own evaluation order (detector.py:383-418): union entries keyed by
// (row, neighbour community), stable-sorted, each group summed with np.add.reduceat's order
// (first + pairwise(rest)), then per row the first maximum over non-own groups in
// ascending community order, taken iff it strictly beats staying.  Bit-identical for any
// real weights and independent of scheduling (the integer paths' atomics are exact only
// for integer sums).

__global__ void k_ps_keys(const int64_t *uptr, const int32_t *unbr, const double *uu,
                          const int32_t *lab, int64_t n, int bc, uint64_t *keys, double *vals) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < n; r += nw)
        for (int64_t e = uptr[r] + lane; e < uptr[r + 1]; e += 32) {
            keys[e] = ((uint64_t)r << bc) | (uint32_t)lab[unbr[e]];
            vals[e] = uu[e];
        }
}
__global__ void k_ps_heads(const uint64_t *keys, int64_t E, int64_t *head) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x)
        head[e] = (e == 0 || keys[e] != keys[e - 1]) ? 1 : 0;
}
__global__ void k_ps_groups(const uint64_t *keys, const int64_t *head, const int64_t *gid,
                            int64_t E, int64_t *gstart, uint64_t *gkey) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x)
        if (head[e]) {
            gstart[gid[e]] = e;
            gkey[gid[e]] = keys[e];
        }
}
__global__ void k_ps_sums(const double *vals, const int64_t *gstart, int64_t ng, int64_t E,
                          double *gsum) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = gstart[g], b = g + 1 < ng ? gstart[g + 1] : E;
        gsum[g] = reduceat_seq(vals + a, b - a);
    }
}
// first group of every row (groups are ordered by row): lower bound of r << bc
__global__ void k_ps_rowptr(const uint64_t *gkey, int64_t ng, int64_t n, int bc, int64_t *rp) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = (uint64_t)r << bc;
        int64_t lo = 0, hi = ng;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (gkey[mid] < k) lo = mid + 1;
            else hi = mid;
        }
        rp[r] = lo;
    }
}
__global__ void k_ps_select(PlanArgs A, const uint64_t *gkey, const double *gsum,
                            const int64_t *rp, int64_t n, uint64_t cmask) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < n; r += nw) {
        const int32_t L = A.label[r];
        const double so = A.s_out[r], si = A.s_in[r];
        double bt = -INFINITY, tstay = 0.0;
        int32_t bc = 0x7fffffff;
        int hown = 0;
        for (int64_t g = rp[r] + lane; g < rp[r + 1]; g += 32) {
            const int32_t c = (int32_t)(gkey[g] & cmask);
            const bool own = c == L;
            const double t = plan_gain(gsum[g], own, so, si, A.S_in[c], A.S_out[c], A.m, A.m2);
            if (own) {
                tstay = t;
                hown = 1;
            } else if (better(t, c, bt, bc)) {
                bt = t;
                bc = c;
            }
        }
        warp_argmax(bt, bc);
        const unsigned om = __ballot_sync(0xffffffffu, hown);
        tstay = __shfl_sync(0xffffffffu, tstay, om ? __ffs(om) - 1 : 0);
        if (lane == 0) {
            if (!om) tstay = -(so * (A.S_in[L] - si) + si * (A.S_out[L] - so)) / A.m2;
            A.cstar[r] = (bc != 0x7fffffff && bt > tstay) ? bc : L;
        }
    }
}

static void run_plan_sorted(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m,
                            int32_t *d_cstar, unsigned long long *d_groups) {
    cudaStream_t s = ctx->stream;
    const int64_t n = G.n, E = G.ue;
    PlanArgs A = make_args(G, F, m, d_cstar);
    const int bc = bits_for(F.n_comms + 1);
    CTX_SCRATCH(DBuf<uint64_t>, pkeys);
    CTX_SCRATCH(DBuf<double>, pvals);
    CTX_SCRATCH(DBuf<int64_t>, phead);
    CTX_SCRATCH(DBuf<int64_t>, pgid);
    pkeys.resize(E);
    pvals.resize(E);
    phead.resize(E + 1);
    pgid.resize(E + 1);
    if (E) {
        k_ps_keys<<<grid_for(n * 32, 256), 256, 0, s>>>(G.uptr.p, G.unbr.p, G.uu.p, F.comm.p, n, bc,
                                                        pkeys.p, pvals.p);
        sort_pairs_u64_f64(ctx, pkeys, pvals, E, bits_for(n + 1) + bc);
        k_ps_heads<<<grid_for(E, 256), 256, 0, s>>>(pkeys.p, E, phead.p);
    }
    CUDA_TRY(cudaMemsetAsync(phead.p + E, 0, 8, s));
    dev_exclusive_sum<int64_t, int64_t>(ctx, phead.p, pgid.p, E + 1);
    int64_t ng = 0;
    CUDA_TRY(cudaMemcpyAsync(&ng, pgid.p + E, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    DBuf<int64_t> gstart, rp;
    DBuf<uint64_t> gkey;
    DBuf<double> gsum;
    gstart.resize(ng);
    gkey.resize(ng);
    gsum.resize(ng);
    rp.resize(n + 1);
    if (ng) {
        k_ps_groups<<<grid_for(E, 256), 256, 0, s>>>(pkeys.p, phead.p, pgid.p, E, gstart.p, gkey.p);
        k_ps_sums<<<grid_for(ng, 128), 128, 0, s>>>(pvals.p, gstart.p, ng, E, gsum.p);
    }
    k_ps_rowptr<<<grid_for(n + 1, 256), 256, 0, s>>>(gkey.p, ng, n, bc, rp.p);
    if (n) k_ps_select<<<grid_for(n * 32, 256), 256, 0, s>>>(A, gkey.p, gsum.p, rp.p, n,
                                                             (1ull << bc) - 1);
    if (d_groups && ng) {
        const unsigned long long g64 = (unsigned long long)ng;
        CUDA_TRY(cudaMemcpyAsync(d_groups, &g64, 8, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
    CUDA_TRY(cudaGetLastError());
}

void run_plan(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m, int32_t *d_cstar,
              int bin_mask, unsigned long long *d_groups) {
    static const bool force_sorted = getenv("SLM_PLAN_SORTED") != nullptr;
    static const bool force_generic = getenv("SLM_FORCE_GENERIC") != nullptr;
    if (G.u32_ok && !force_generic && !force_sorted) {
        run_plan_u32(ctx, G, F, m, d_cstar, bin_mask, d_groups);
        return;
    }
    if ((!G.integral || force_sorted) && bin_mask == 127) {
        // real-valued weights: the reference's stable-sort + reduceat order (deterministic)
        run_plan_sorted(ctx, G, F, m, d_cstar, d_groups);
        return;
    }
    // generic fp64 path (non-integer weights or row totals >= 2^32)
    cudaStream_t s = ctx->stream;
    int64_t n = G.n;
    // rows without entries keep their label (detector.py:379-382)
    if (bin_mask & 64) k_copy_labels<<<grid_for(n, 256), 256, 0, s>>>(F.comm.p, n, d_cstar);
    PlanArgs A = make_args(G, F, m, d_cstar);
    A.groups = d_groups;
    int64_t ns = G.bin_off[1] - G.bin_off[0];
    int64_t nm = G.bin_off[4] - G.bin_off[1];
    int64_t nl = G.bin_off[6] - G.bin_off[4];
    if (ns && (bin_mask & 1))
        k_plan_small<<<grid_for(ns * 32, 256, SMS() * 64), 256, 0, s>>>(A, G.bin_rows.p + G.bin_off[0], ns);
    if (nm && (bin_mask & 14)) {
        size_t sm = MID_H * (sizeof(double) + sizeof(int32_t));
        CUDA_TRY(cudaFuncSetAttribute(k_plan_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_plan_mid<<<(unsigned)std::min<int64_t>(nm, SMS() * 2 * 8), MID_BLOCK, sm, s>>>(A, G.bin_rows.p + G.bin_off[1], nm);
    }
    if (nl && (bin_mask & 48)) {
        ctx->hash_keys.resize(G.large_hash_total);
        ctx->hash_vals.resize(G.large_hash_total);
        k_plan_large<<<(unsigned)std::min<int64_t>(nl, SMS() * 2), LARGE_BLOCK, 0, s>>>(
            A, G.bin_rows.p + G.bin_off[4], nl, G.large_hoff.p, ctx->hash_keys.p, ctx->hash_vals.p);
    }
    CUDA_TRY(cudaGetLastError());
}

// ------------------------------------------------------------------ ASSIGN

__global__ void __launch_bounds__(256) k_assign(const int64_t *uptr, const int32_t *unbr,
                                                const double *uu, const double *s_out,
                                                const double *s_in, int64_t n, double m, double m2,
                                                int32_t *a) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w; r < n; r += nw) {
        const int64_t e0 = uptr[r], e1 = uptr[r + 1];
        const double so = s_out[r], si = s_in[r];
        double bt = -INFINITY;
        int64_t be = INT64_MAX;
        for (int64_t e = e0 + lane; e < e1; e += 32) {
            int32_t j = unbr[e];
            double g = uu[e] / m - (so * s_in[j] + si * s_out[j]) / m2;
            if (g > bt) {   // lanes visit ascending e: first max per lane kept
                bt = g;
                be = e;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            double ot = __shfl_xor_sync(0xffffffffu, bt, off);
            int64_t oe = __shfl_xor_sync(0xffffffffu, be, off);
            if (ot > bt || (ot == bt && oe < be)) {
                bt = ot;
                be = oe;
            }
        }
        if (lane == 0) a[r] = (e1 > e0 && bt > 0.0) ? unbr[be] : (int32_t)r;
    }
}

void run_assign(slm_ctx *ctx, const LevelGraph &G, double m, int32_t *d_a) {
    int64_t n = G.n;
    k_assign<<<grid_for(n * 32, 256, SMS() * 64), 256, 0, ctx->stream>>>(
        G.uptr.p, G.unbr.p, G.uu.p, G.s_out.p, G.s_in.p, n, m, m * m, d_a);
    CUDA_TRY(cudaGetLastError());
}

// ------------------------------------------------------------- LOCAL GAINS

__global__ void __launch_bounds__(256) k_local_gains(const int64_t *uptr, const int32_t *unbr,
                                                     const double *uu, const int32_t *label,
                                                     const double *S_out, const double *S_in,
                                                     const double *s_out, const double *s_in,
                                                     int64_t n, double m, double *lg,
                                                     uint8_t *bad) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w; r < n; r += nw) {
        const int32_t L = label[r];
        double own = 0.0;
        for (int64_t e = uptr[r] + lane; e < uptr[r + 1]; e += 32)
            if (label[unbr[e]] == L) own += uu[e];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) own += __shfl_xor_sync(0xffffffffu, own, off);
        if (lane == 0) {
            const double so = s_out[r], si = s_in[r];
            double g = own / m - (so * (S_in[L] - si) + si * (S_out[L] - so)) / (m * m);
            if (m == 0.0) g = 0.0;
            if (lg) lg[r] = g;
            if (g < 0.0) bad[L] = 1;
        }
    }
}

void run_local_gains_u32(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m, double *d_lg,
                         uint8_t *d_bad);

void run_local_gains(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m, double *d_lg,
                     uint8_t *d_bad) {
    int64_t n = G.n;
    if (G.u32_ok) {
        run_local_gains_u32(ctx, G, F, m, d_lg, d_bad);
        return;
    }
    k_local_gains<<<grid_for(n * 32, 256, SMS() * 64), 256, 0, ctx->stream>>>(
        G.uptr.p, G.unbr.p, G.uu.p, F.comm.p, F.S_out.p, F.S_in.p, G.s_out.p, G.s_in.p, n, m,
        d_lg, d_bad);
    CUDA_TRY(cudaGetLastError());
}

// a kernel of this translation unit (module preloading, slm_capi.cu preload_modules)
const void *slm_anchor_plan() { return (const void *)k_assign; }
