// slm_commit.cu -- MAXIMAL correction commit (maximal_correction, detector.py:457-521).
//
// The reference commits the planned moves serially in ascending node id: a candidate is
// skipped once its source community is dirty, needs a passing coin (rng.py:34-43), a
// non-empty target, a strictly positive re-priced gain (gain_switch, quality.py:186-219) and
// an attach target (detector.py:440-454); a commit drags the node's assignment tail
// (detector.py:421-437) into the target community.
//
// Exact parallel replay by rounds.  A candidate's outcome depends on earlier commits only
// through its two communities.  Each round evaluates every unresolved candidate against
// the live state ("tentative outcome"), then computes by fixpoint the set of candidates that
// an earlier *possible* commit could still influence (sharing a community with an earlier
// tentative commit, transitively); every other candidate's tentative outcome is final.
// Final commits of one round are pairwise community-disjoint, so they apply in parallel
// with plain stores.  The earliest unresolved candidate is always final, so rounds make
// progress; rounds track chains of dependent *commits*, not of skips.
//
// Tails are contiguous ranges of the community DFS layout (slm_forest.cu): a cycle node's
// tail is its whole community, any other node's tail is its DFS subtree.
#include "slm_internal.cuh"
#include <cub/cub.cuh>

#define GS_LOOP(i, n)                                                                      \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n);              \
         i += (int64_t)gridDim.x * blockDim.x)

struct CandSpec {
    double w_to, w_from, so_b, si_b;
    int32_t j;
    int32_t tail_lo, tail_hi;   // range in F.order
    int32_t pad;
};

enum { ST_UNRES = 0, ST_SKIP = 1, ST_COMMIT = 2, ST_COIN = 3 };

__global__ void k_cand_flags(const int32_t *cstar, const int32_t *comm, int64_t n, int32_t *f) {
    GS_LOOP(i, n) f[i] = (cstar[i] != comm[i]) ? 1 : 0;
}
__global__ void k_cand_scatter(const int32_t *f, const int32_t *pos, int64_t n, int32_t *cand) {
    GS_LOOP(i, n) if (f[i]) cand[pos[i]] = (int32_t)i;
}

__global__ void k_coins(const int32_t *cand, int64_t K, uint64_t base, double p, uint8_t *status) {
    GS_LOOP(k, K) status[k] = (uniform01_at(base, cand[k]) < p) ? ST_UNRES : ST_COIN;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// w_to (live labels) over the tail, and the attach target of i in `to` (detector.py:440-454)
__device__ void eval_to_side(const int64_t *uptr, const int32_t *unbr, const double *uu,
                             const double *s_out, const double *s_in, const int32_t *lab,
                             const int32_t *order, int32_t lo, int32_t hi, int32_t i, int32_t to,
                             double m, double m2, double &w_to, int32_t &j) {
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    for (int32_t q = lo; q < hi; q++) {
        int32_t x = order[q];
        for (int64_t e = uptr[x] + lane; e < uptr[x + 1]; e += 32)
            if (lab[unbr[e]] == to) acc += uu[e];
    }
    w_to = warp_sum(acc);
    const double soi = s_out[i], sii = s_in[i];
    double bt = -INFINITY;
    int64_t be = INT64_MAX;
    for (int64_t e = uptr[i] + lane; e < uptr[i + 1]; e += 32) {
        int32_t z = unbr[e];
        if (lab[z] != to) continue;
        double pg = uu[e] / m - (soi * s_in[z] + sii * s_out[z]) / m2;
        if (pg > bt) {
            bt = pg;
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
    j = (be != INT64_MAX) ? unbr[be] : -1;
}

struct CommitArgs {
    const int64_t *uptr;
    const int32_t *unbr;
    const double *uu;
    const double *s_out, *s_in;
    const int32_t *comm;      // snapshot labels
    const uint8_t *on_cycle;
    const int32_t *cptr, *order, *pos, *sz;
    const int32_t *cand, *cstar;
    double m, m2;
};

// speculative evaluation against the snapshot (one warp per accepted candidate)
__global__ void k_spec(CommitArgs A, int64_t K, const uint8_t *status, CandSpec *spec) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = w; k < K; k += nw) {
        if (status[k] != ST_UNRES) continue;
        const int32_t i = A.cand[k];
        const int32_t frm = A.comm[i], to = A.cstar[i];
        const int32_t base = A.cptr[frm];
        int32_t lo, hi;
        if (A.on_cycle[i]) {
            lo = base;
            hi = A.cptr[frm + 1];
        } else {
            lo = base + A.pos[i];
            hi = lo + A.sz[i];
        }
        const int32_t plo = lo - base, phi = hi - base;
        double so = 0.0, si = 0.0, wf = 0.0;
        for (int32_t q = lo + lane; q < hi; q += 32) {
            int32_t x = A.order[q];
            so += A.s_out[x];
            si += A.s_in[x];
        }
        for (int32_t q = lo; q < hi; q++) {
            int32_t x = A.order[q];
            for (int64_t e = A.uptr[x] + lane; e < A.uptr[x + 1]; e += 32) {
                int32_t z = A.unbr[e];
                if (A.comm[z] != frm) continue;
                int32_t pz = A.pos[z];
                if (pz >= plo && pz < phi) continue;   // z inside the moved tail
                wf += A.uu[e];
            }
        }
        so = warp_sum(so);
        si = warp_sum(si);
        wf = warp_sum(wf);
        double wt;
        int32_t j;
        eval_to_side(A.uptr, A.unbr, A.uu, A.s_out, A.s_in, A.comm, A.order, lo, hi, i, to, A.m,
                     A.m2, wt, j);
        if (lane == 0) {
            CandSpec c;
            c.w_to = wt;
            c.w_from = wf;
            c.so_b = so;
            c.si_b = si;
            c.j = j;
            c.tail_lo = lo;
            c.tail_hi = hi;
            c.pad = 0;
            spec[k] = c;
        }
    }
}

struct LiveState {
    int32_t *lab;
    double *S_out, *S_in;
    int32_t *cnt;
    uint8_t *dirty;
    int32_t *first_commit;
    int32_t *a;
};

// tentative evaluation of every unresolved candidate against the live state
__global__ void k_tentative(CommitArgs A, LiveState S, int64_t K, uint8_t *status,
                            const CandSpec *spec, uint8_t *tent, double *tgain, int32_t *tj) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = w; k < K; k += nw) {
        if (status[k] != ST_UNRES) continue;
        const int32_t i = A.cand[k];
        const int32_t frm = A.comm[i], to = A.cstar[i];
        if (S.dirty[frm]) {                 // detector.py:489-490
            if (lane == 0) status[k] = ST_SKIP;
            continue;
        }
        const CandSpec c = spec[k];
        double wt = c.w_to;
        int32_t j = c.j;
        bool ok = S.cnt[to] != 0;           // detector.py:494-495
        if (ok && S.dirty[to])
            eval_to_side(A.uptr, A.unbr, A.uu, A.s_out, A.s_in, S.lab, A.order, c.tail_lo,
                         c.tail_hi, i, to, A.m, A.m2, wt, j);
        if (lane == 0) {
            double g = 0.0;
            if (ok) {
                const double so_b = c.so_b, si_b = c.si_b;
                const double so_t = S.S_out[to], si_t = S.S_in[to];
                // gain_switch d_null, quality.py:216-219, exact operand order
                double d_null = -S.S_out[frm] * si_b - so_b * S.S_in[frm] + so_t * si_b +
                                so_b * si_t + 2.0 * so_b * si_b;
                g = (wt - c.w_from) / A.m - d_null / (A.m * A.m);
                ok = (g > 0.0) && (j >= 0);  // detector.py:498-502
            }
            tent[k] = ok ? 1 : 0;
            tgain[k] = g;
            tj[k] = j;
        }
    }
}

__global__ void k_src_init(int64_t K, const uint8_t *status, const uint8_t *tent, uint8_t *srcf) {
    GS_LOOP(k, K) srcf[k] = (status[k] == ST_UNRES && tent[k]) ? 1 : 0;
}
__global__ void k_minsrc_reset(const int32_t *cand, const int32_t *comm, const int32_t *cstar,
                               int64_t K, const uint8_t *status, int32_t *minsrc) {
    GS_LOOP(k, K) {
        if (status[k] != ST_UNRES) continue;
        int32_t i = cand[k];
        minsrc[comm[i]] = 0x7fffffff;
        minsrc[cstar[i]] = 0x7fffffff;
    }
}
__global__ void k_minsrc(const int32_t *cand, const int32_t *comm, const int32_t *cstar, int64_t K,
                         const uint8_t *status, const uint8_t *srcf, int32_t *minsrc) {
    GS_LOOP(k, K) {
        if (status[k] != ST_UNRES || !srcf[k]) continue;
        int32_t i = cand[k];
        atomicMin(&minsrc[comm[i]], (int32_t)k);
        atomicMin(&minsrc[cstar[i]], (int32_t)k);
    }
}
__global__ void k_unstable_update(const int32_t *cand, const int32_t *comm, const int32_t *cstar,
                                  int64_t K, const uint8_t *status, const uint8_t *tent,
                                  const int32_t *minsrc, uint8_t *srcf, uint8_t *unst,
                                  int32_t *changed) {
    GS_LOOP(k, K) {
        if (status[k] != ST_UNRES) continue;
        int32_t i = cand[k];
        bool u = minsrc[comm[i]] < (int32_t)k || minsrc[cstar[i]] < (int32_t)k;
        unst[k] = u;
        uint8_t sf = (tent[k] || u) ? 1 : 0;
        if (sf != srcf[k]) {
            srcf[k] = sf;
            *changed = 1;
        }
    }
}

// apply final outcomes: stable tentative commits commit, stable skips resolve
__global__ void k_apply(CommitArgs A, LiveState S, int64_t K, uint8_t *status, const uint8_t *tent,
                        const uint8_t *unst, const CandSpec *spec, const int32_t *tj,
                        int32_t *remaining) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = w; k < K; k += nw) {
        if (status[k] != ST_UNRES) continue;
        if (unst[k]) {
            if (lane == 0) atomicAdd(remaining, 1);
            continue;
        }
        if (!tent[k]) {
            if (lane == 0) status[k] = ST_SKIP;
            continue;
        }
        const int32_t i = A.cand[k];
        const int32_t frm = A.comm[i], to = A.cstar[i];
        const CandSpec c = spec[k];
        for (int32_t q = c.tail_lo + lane; q < c.tail_hi; q += 32) S.lab[A.order[q]] = to;
        if (lane == 0) {
            S.a[i] = tj[k];
            // move_nodes (quality.py:87-95)
            S.S_out[frm] -= c.so_b;
            S.S_in[frm] -= c.si_b;
            S.cnt[frm] -= (c.tail_hi - c.tail_lo);
            S.S_out[to] += c.so_b;
            S.S_in[to] += c.si_b;
            S.cnt[to] += (c.tail_hi - c.tail_lo);
            S.dirty[frm] = 1;
            S.dirty[to] = 1;
            atomicMin(&S.first_commit[frm], (int32_t)k);
            atomicMin(&S.first_commit[to], (int32_t)k);
            status[k] = ST_COMMIT;
        }
    }
}

__global__ void k_coin_blocked(const int32_t *cand, const int32_t *comm, int64_t K,
                               const uint8_t *status, const int32_t *first_commit,
                               int32_t *out) {
    GS_LOOP(k, K) {
        if (status[k] != ST_COIN) continue;
        // reached (frm clean at k) and lost the coin: detector.py:489-493
        if (first_commit[comm[cand[k]]] > (int32_t)k) atomicOr(&out[0], 1);
    }
}

__global__ void k_commit_flags(int64_t K, const uint8_t *status, int32_t *f) {
    GS_LOOP(k, K) f[k] = status[k] == ST_COMMIT ? 1 : 0;
}
__global__ void k_gather_gains(int64_t K, const int32_t *f, const int32_t *pos, const double *g,
                               double *out) {
    GS_LOOP(k, K) if (f[k]) out[pos[k]] = g[k];
}

void run_commit(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m, const int32_t *d_cstar,
                uint64_t seed, double accept_prob, int64_t level, int64_t sweep, int *improved,
                int64_t *applied, std::vector<double> *gains) {
    cudaStream_t s = ctx->stream;
    const int64_t n = G.n, nc = F.n_comms;
    *improved = 0;
    *applied = 0;
    ctx->last_rounds = 0;
    // candidates: cstar != label, ascending (detector.py:473)
    DBuf<int32_t> flag, pos, cand;
    flag.resize(n + 1);
    pos.resize(n + 1);
    CUDA_TRY(cudaMemsetAsync(flag.p + n, 0, 4, s));
    k_cand_flags<<<grid_for(n, 256), 256, 0, s>>>(d_cstar, F.comm.p, n, flag.p);
    cub_exclusive_sum<int32_t>(ctx, flag.p, pos.p, n + 1);
    int32_t K = 0;
    CUDA_TRY(cudaMemcpyAsync(&K, pos.p + n, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    ctx->last_candidates = K;
    if (K == 0) return;
    cand.resize(K);
    k_cand_scatter<<<grid_for(n, 256), 256, 0, s>>>(flag.p, pos.p, n, cand.p);
    DBuf<uint8_t> status, tent, srcf, unst;
    status.resize(K);
    tent.resize(K);
    srcf.resize(K);
    unst.resize(K);
    k_coins<<<grid_for(K, 256), 256, 0, s>>>(cand.p, K, mix_key2(seed, level, sweep), accept_prob,
                                             status.p);
    CommitArgs A;
    A.uptr = G.uptr.p;
    A.unbr = G.unbr.p;
    A.uu = G.uu.p;
    A.s_out = G.s_out.p;
    A.s_in = G.s_in.p;
    A.comm = F.comm.p;
    A.on_cycle = F.on_cycle.p;
    A.cptr = F.cptr.p;
    A.order = F.order.p;
    A.pos = F.pos.p;
    A.sz = F.sz.p;
    A.cand = cand.p;
    A.cstar = d_cstar;
    A.m = m;
    A.m2 = m * m;
    DBuf<CandSpec> spec;
    spec.resize(K);
    unsigned GW = grid_for((int64_t)K * 32, 256, 148LL * 32);
    k_spec<<<GW, 256, 0, s>>>(A, K, status.p, spec.p);
    // live state
    DBuf<int32_t> lab, cnt, first_commit, minsrc, tj;
    DBuf<double> So, Si, tgain;
    DBuf<uint8_t> dirty;
    lab.resize(n);
    cnt.resize(nc);
    first_commit.resize(nc);
    minsrc.resize(nc);
    So.resize(nc);
    Si.resize(nc);
    dirty.resize(nc);
    tgain.resize(K);
    tj.resize(K);
    CUDA_TRY(cudaMemcpyAsync(lab.p, F.comm.p, n * 4, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(cnt.p, F.count.p, nc * 4, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(So.p, F.S_out.p, nc * 8, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(Si.p, F.S_in.p, nc * 8, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemsetAsync(dirty.p, 0, nc, s));
    CUDA_TRY(cudaMemsetAsync(first_commit.p, 0x7f, nc * 4, s));   // 0x7f7f7f7f > any k
    LiveState S;
    S.lab = lab.p;
    S.S_out = So.p;
    S.S_in = Si.p;
    S.cnt = cnt.p;
    S.dirty = dirty.p;
    S.first_commit = first_commit.p;
    S.a = F.a.p;   // committed pointers are written in place (forest.a copy semantics:
                   // the static tails come from the layout built before this call)
    int32_t *dflags = ctx->i32d.resize(4);
    unsigned GK = grid_for(K, 256);
    for (int round = 0;; round++) {
        k_tentative<<<GW, 256, 0, s>>>(A, S, K, status.p, spec.p, tent.p, tgain.p, tj.p);
        k_src_init<<<GK, 256, 0, s>>>(K, status.p, tent.p, srcf.p);
        for (int it = 0;; it++) {
            k_minsrc_reset<<<GK, 256, 0, s>>>(cand.p, F.comm.p, d_cstar, K, status.p, minsrc.p);
            k_minsrc<<<GK, 256, 0, s>>>(cand.p, F.comm.p, d_cstar, K, status.p, srcf.p, minsrc.p);
            CUDA_TRY(cudaMemsetAsync(dflags, 0, 4, s));
            k_unstable_update<<<GK, 256, 0, s>>>(cand.p, F.comm.p, d_cstar, K, status.p, tent.p,
                                                 minsrc.p, srcf.p, unst.p, dflags);
            int32_t ch = 0;
            CUDA_TRY(cudaMemcpyAsync(&ch, dflags, 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            if (!ch) break;
        }
        CUDA_TRY(cudaMemsetAsync(dflags + 1, 0, 4, s));
        k_apply<<<GW, 256, 0, s>>>(A, S, K, status.p, tent.p, unst.p, spec.p, tj.p, dflags + 1);
        int32_t rem = 0;
        CUDA_TRY(cudaMemcpyAsync(&rem, dflags + 1, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        ctx->last_rounds = round + 1;
        if (rem == 0) break;
    }
    CUDA_TRY(cudaMemsetAsync(dflags + 2, 0, 4, s));
    k_coin_blocked<<<GK, 256, 0, s>>>(cand.p, F.comm.p, K, status.p, first_commit.p, dflags + 2);
    // applied + gains in ascending candidate order
    DBuf<int32_t> cf, cpos;
    cf.resize(K + 1);
    cpos.resize(K + 1);
    CUDA_TRY(cudaMemsetAsync(cf.p + K, 0, 4, s));
    k_commit_flags<<<GK, 256, 0, s>>>(K, status.p, cf.p);
    cub_exclusive_sum<int32_t>(ctx, cf.p, cpos.p, K + 1);
    int32_t hv[2] = {0, 0};
    CUDA_TRY(cudaMemcpyAsync(&hv[0], cpos.p + K, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&hv[1], dflags + 2, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *applied = hv[0];
    *improved = (hv[0] > 0) || hv[1];
    if (gains && hv[0] > 0) {
        DBuf<double> gg;
        gg.resize(hv[0]);
        k_gather_gains<<<GK, 256, 0, s>>>(K, cf.p, cpos.p, tgain.p, gg.p);
        gains->resize(hv[0]);
        CUDA_TRY(cudaMemcpyAsync(gains->data(), gg.p, hv[0] * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
}
