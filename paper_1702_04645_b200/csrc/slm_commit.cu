// slm_commit.cu -- MAXIMAL correction commit (maximal_correction, detector.py:457-521).
//
// The reference commits the planned moves serially in ascending node id: a candidate is
// skipped once its source community is dirty, needs a passing coin (rng.py:34-43), a
// non-empty target, a strictly positive re-priced gain (gain_switch, quality.py:186-219) and
// an attach target (detector.py:440-454); a commit drags the node's assignment tail
// (detector.py:421-437) into the target community.
//
// Exact parallel replay by community timelines.  A candidate's outcome depends on earlier
// commits only through its two communities (frm, to).  Every community C gets the ordered
// list of accepted candidates touching it (its timeline) and one warp that walks it: the
// walker evaluates the candidates that move INTO C (C owns its target-side state: S[C],
// count[C], labels of nodes moving in), and parks at a candidate that moves OUT of C until
// that candidate's target walker has evaluated it.  Evaluating candidate k therefore only
// waits for frm_k's walker to have reached k -- so a long chain of candidates into one hub
// community is walked in a single pass, with per-candidate data prefetched 32 at a time.
// Rounds (kernel relaunches) hand parked walkers over; the earliest unresolved candidate is
// always evaluable, so every round makes progress.  Candidates whose tail has no neighbour
// that can move keep their snapshot w_to / attach target even when `to` has changed
// (only S[to] is re-read); the others are re-priced against the live labels.
//
// Tails are contiguous ranges of the community DFS layout (slm_forest.cu): a cycle node's
// tail is its whole community, any other node's tail is its DFS subtree.
#include "slm_internal.cuh"
#include <string>

#define GS_LOOP(i, n)                                                                      \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n);              \
         i += (int64_t)gridDim.x * blockDim.x)

struct CandSpec {
    double w_to, w_from, so_b, si_b;
    double pgj;          // pairwise gain of the snapshot attach target j
    int64_t je;          // its union entry index (row order = tie-break order), -1 if none
    int64_t mv_off;      // moving-neighbour entries of the tail: [mv_off, mv_off + mv_cnt)
    int32_t j;
    int32_t tail_lo, tail_hi;   // range in F.order
    int32_t mv_cnt;
};

enum { ST_UNRES = 0, ST_SKIP = 1, ST_COMMIT = 2, ST_COIN = 3 };

__global__ void k_cand_flags(const int32_t *cstar, const int32_t *comm, int64_t n, int32_t *f) {
    GS_LOOP(i, n) f[i] = (cstar[i] != comm[i]) ? 1 : 0;
}
__global__ void k_cand_scatter(const int32_t *f, const int32_t *pos, int64_t n, int32_t *cand) {
    GS_LOOP(i, n) if (f[i]) cand[pos[i]] = (int32_t)i;
}

__global__ void k_coins(const int32_t *cand, int64_t K, uint64_t base, double p, int32_t *status) {
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
                             double m, double m2, double &w_to, int32_t &j, int64_t *je = nullptr,
                             double *pgj = nullptr) {
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
    if (je) *je = (be != INT64_MAX) ? be : -1;
    if (pgj) *pgj = bt;
}

// attach target of i among the entries of its own row only (live labels)
__device__ void attach_only(const int64_t *uptr, const int32_t *unbr, const double *uu,
                            const double *s_out, const double *s_in, const int32_t *lab, int32_t i,
                            int32_t to, double m, double m2, int32_t &j) {
    const int lane = threadIdx.x & 31;
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
    int runs;                 // run commits after a commit (walk_run; SLM_WALK_RUNS=0 disables)
};

// candidates whose tail has more members than this, or whose tail rows hold more union
// entries than BIG_VOL (coarse-level hubs), are evaluated by a whole CTA
constexpr int BIG_TAIL = 64;
constexpr int64_t BIG_VOL = 4096;

__device__ __forceinline__ void tail_range(const CommitArgs &A, int32_t i, int32_t frm, int32_t &lo,
                                           int32_t &hi) {
    const int32_t base = A.cptr[frm];
    if (A.on_cycle[i]) {
        lo = base;
        hi = A.cptr[frm + 1];
    } else {
        lo = base + A.pos[i];
        hi = lo + A.sz[i];
    }
}

// speculative evaluation against the snapshot (one warp per accepted candidate; tails of
// more than BIG_TAIL members are listed for k_spec_big)
__global__ void k_spec(CommitArgs A, int64_t K, const int32_t *status, CandSpec *spec,
                       int32_t *big, int32_t *nbig, int64_t *vol_out, int64_t big_vol) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = w; k < K; k += nw) {
        if (status[k] != ST_UNRES) continue;
        const int32_t i = A.cand[k];
        const int32_t frm = A.comm[i], to = A.cstar[i];
        const int32_t base = A.cptr[frm];
        int32_t lo, hi;
        tail_range(A, i, frm, lo, hi);
        bool isbig = hi - lo > BIG_TAIL;
        if (!isbig) {
            int64_t vol = 0;
            for (int32_t q = lo + lane; q < hi; q += 32) {
                const int32_t x = A.order[q];
                vol += A.uptr[x + 1] - A.uptr[x];
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) vol += __shfl_xor_sync(0xffffffffu, vol, off);
            isbig = vol > big_vol;
            if (lane == 0) vol_out[k] = vol;   // capacity of its moving-neighbour list
        }
        if (isbig) {
            if (lane == 0) big[atomicAdd(nbig, 1)] = (int32_t)k;
            continue;
        }
        const int32_t plo = lo - base, phi = hi - base;
        double so = 0.0, si = 0.0, wf = 0.0, wt = 0.0;
        for (int32_t q = lo + lane; q < hi; q += 32) {
            int32_t x = A.order[q];
            so += A.s_out[x];
            si += A.s_in[x];
        }
        // one pass over the tail rows: w_from, w_to, and on row i the attach target
        // (detector.py:440-454: first maximum in entry order)
        const double soi = A.s_out[i], sii = A.s_in[i];
        double bt = -INFINITY;
        int64_t be = INT64_MAX;
        for (int32_t q = lo; q < hi; q++) {
            const int32_t x = A.order[q];
            const bool xi = x == i;
            for (int64_t e = A.uptr[x] + lane; e < A.uptr[x + 1]; e += 32) {
                const int32_t z = A.unbr[e];
                const int32_t cz = A.comm[z];
                if (cz == to) {
                    const double u = A.uu[e];
                    wt += u;
                    if (xi) {
                        const double pg = u / A.m - (soi * A.s_in[z] + sii * A.s_out[z]) / A.m2;
                        if (pg > bt) {
                            bt = pg;
                            be = e;
                        }
                    }
                }
                if (cz != frm) continue;
                int32_t pz = A.pos[z];
                if (pz >= plo && pz < phi) continue;   // z inside the moved tail
                wf += A.uu[e];
            }
        }
        so = warp_sum(so);
        si = warp_sum(si);
        wf = warp_sum(wf);
        wt = warp_sum(wt);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ot = __shfl_xor_sync(0xffffffffu, bt, off);
            const int64_t oe = __shfl_xor_sync(0xffffffffu, be, off);
            if (ot > bt || (ot == bt && oe < be)) {
                bt = ot;
                be = oe;
            }
        }
        const double pgj = bt;
        const int32_t j = be != INT64_MAX ? A.unbr[be] : -1;
        const int64_t je = be != INT64_MAX ? be : -1;
        if (lane == 0) {
            CandSpec c;
            c.w_to = wt;
            c.w_from = wf;
            c.so_b = so;
            c.si_b = si;
            c.pgj = pgj;
            c.je = je;
            c.mv_off = 0;
            c.j = j;
            c.tail_lo = lo;
            c.tail_hi = hi;
            c.mv_cnt = 0;
            spec[k] = c;
        }
    }
}


// one CTA per big-tail candidate: the tail's strengths, w_from and w_to by all warps
// (members over warps, entries over lanes), the attach target over row i by warp 0
constexpr int SPEC_BLOCK = 512;
__global__ void __launch_bounds__(SPEC_BLOCK) k_spec_big(CommitArgs A, const int32_t *big,
                                                         const int32_t *nbig, CandSpec *spec,
                                                         int64_t *vol_out) {
    __shared__ double red[4][SPEC_BLOCK / 32];
    __shared__ unsigned long long s_vol;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = SPEC_BLOCK / 32;
    const int32_t nb = *nbig;
    for (int32_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const int32_t k = big[b];
        const int32_t i = A.cand[k];
        const int32_t frm = A.comm[i], to = A.cstar[i];
        const int32_t base = A.cptr[frm];
        int32_t lo, hi;
        tail_range(A, i, frm, lo, hi);
        const int32_t plo = lo - base, phi = hi - base;
        double so = 0.0, si = 0.0, wf = 0.0, wt = 0.0;
        if (threadIdx.x == 0) s_vol = 0;
        __syncthreads();
        unsigned long long vol = 0;
        for (int32_t q = lo + threadIdx.x; q < hi; q += SPEC_BLOCK) {
            const int32_t x = A.order[q];
            so += A.s_out[x];
            si += A.s_in[x];
            vol += (unsigned long long)(A.uptr[x + 1] - A.uptr[x]);
        }
        atomicAdd(&s_vol, vol);
        for (int32_t q = lo + wid; q < hi; q += NW) {
            const int32_t x = A.order[q];
            for (int64_t e = A.uptr[x] + lane; e < A.uptr[x + 1]; e += 32) {
                const int32_t z = A.unbr[e];
                const int32_t cz = A.comm[z];
                if (cz == to) wt += A.uu[e];
                if (cz != frm) continue;
                const int32_t pz = A.pos[z];
                if (pz >= plo && pz < phi) continue;   // z inside the moved tail
                wf += A.uu[e];
            }
        }
        so = warp_sum(so);
        si = warp_sum(si);
        wf = warp_sum(wf);
        wt = warp_sum(wt);
        if (lane == 0) {
            red[0][wid] = so;
            red[1][wid] = si;
            red[2][wid] = wf;
            red[3][wid] = wt;
        }
        __syncthreads();
        if (wid == 0) {
            double v[4];
#pragma unroll
            for (int f = 0; f < 4; f++) v[f] = warp_sum(lane < NW ? red[f][lane] : 0.0);
            // attach target of i in `to` over i's row (detector.py:440-454)
            const double soi = A.s_out[i], sii = A.s_in[i];
            double bt = -INFINITY;
            int64_t be = INT64_MAX;
            for (int64_t e = A.uptr[i] + lane; e < A.uptr[i + 1]; e += 32) {
                const int32_t z = A.unbr[e];
                if (A.comm[z] != to) continue;
                const double pg = A.uu[e] / A.m - (soi * A.s_in[z] + sii * A.s_out[z]) / A.m2;
                if (pg > bt) {
                    bt = pg;
                    be = e;
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ot = __shfl_xor_sync(0xffffffffu, bt, off);
                const int64_t oe = __shfl_xor_sync(0xffffffffu, be, off);
                if (ot > bt || (ot == bt && oe < be)) {
                    bt = ot;
                    be = oe;
                }
            }
            if (lane == 0) {
                vol_out[k] = (int64_t)s_vol;   // capacity of its moving-neighbour list
                CandSpec c;
                c.w_to = v[3];
                c.w_from = v[2];
                c.so_b = v[0];
                c.si_b = v[1];
                c.pgj = bt;
                c.je = be != INT64_MAX ? be : -1;
                c.mv_off = 0;
                c.j = be != INT64_MAX ? A.unbr[be] : -1;
                c.tail_lo = lo;
                c.tail_hi = hi;
                c.mv_cnt = -1;   // big: k_mv_scan leaves it to k_mv_scan_big (which sets it)
                spec[k] = c;
            }
        }
        __syncthreads();
    }
}

// mark every node of an accepted candidate's tail (a node that may move this sweep)
__global__ void k_mark_moving(const int32_t *cand, const int32_t *comm, const uint8_t *on_cycle,
                              const int32_t *cptr, const int32_t *pos, const int32_t *sz,
                              const int32_t *order, int64_t K, const int32_t *status,
                              uint8_t *moving) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = w; k < K; k += nw) {
        if (status[k] != ST_UNRES) continue;
        const int32_t i = cand[k], frm = comm[i], base = cptr[frm];
        int32_t lo, hi;
        if (on_cycle[i]) {
            lo = base;
            hi = cptr[frm + 1];
        } else {
            lo = base + pos[i];
            hi = lo + sz[i];
        }
        for (int32_t q = lo + lane; q < hi; q += 32) moving[order[q]] = 1;
    }
}

// moving-neighbour entries of each accepted candidate's tail: entries (x in tail, z) with z
// outside `frm` and in some accepted tail.  Only these can change w_to / the attach target
// when `to` changes during the sweep, so re-pricing is an exact delta over this list.
__global__ void k_mv_scan(CommitArgs A, int64_t K, const int32_t *status, CandSpec *spec,
                          const uint8_t *moving, int fill, int64_t *cnt, int32_t *mv_z,
                          double *mv_u, int64_t *mv_e, uint8_t *mv_i) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = w; k < K; k += nw) {
        if (status[k] != ST_UNRES) continue;
        const int32_t i = A.cand[k], frm = A.comm[i];
        const CandSpec c = spec[k];
        if (c.mv_cnt < 0) continue;   // big candidate: k_mv_scan_big
        int64_t base = fill ? c.mv_off : 0, total = 0;
        for (int32_t q = c.tail_lo; q < c.tail_hi; q++) {
            const int32_t x = A.order[q];
            for (int64_t e0 = A.uptr[x]; e0 < A.uptr[x + 1]; e0 += 32) {
                const int64_t e = e0 + lane;
                bool hit = false;
                int32_t z = 0;
                if (e < A.uptr[x + 1]) {
                    z = A.unbr[e];
                    hit = moving[z] && A.comm[z] != frm;
                }
                const unsigned hm = __ballot_sync(0xffffffffu, hit);
                if (fill && hit) {
                    const int64_t at = base + total + __popc(hm & ((1u << lane) - 1));
                    mv_z[at] = z;
                    mv_u[at] = A.uu[e];
                    mv_e[at] = e;
                    mv_i[at] = (x == i);
                }
                total += __popc(hm);
            }
        }
        if (lane == 0) {
            if (fill) spec[k].mv_cnt = (int32_t)total;
            else cnt[k] = total;
        }
    }
}
// moving-neighbour scan of the big-tail candidates: one CTA each (entries in any order;
// re-pricing breaks ties by entry index)
__global__ void __launch_bounds__(SPEC_BLOCK) k_mv_scan_big(CommitArgs A, const int32_t *big,
                                                            const int32_t *nbig, CandSpec *spec,
                                                            const uint8_t *moving, int fill,
                                                            int64_t *cnt, int32_t *mv_z, double *mv_u,
                                                            int64_t *mv_e, uint8_t *mv_i) {
    __shared__ unsigned long long s_tot;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = SPEC_BLOCK / 32;
    const int32_t nb = *nbig;
    for (int32_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const int32_t k = big[b];
        const int32_t i = A.cand[k], frm = A.comm[i];
        const CandSpec c = spec[k];
        if (threadIdx.x == 0) s_tot = 0;
        __syncthreads();
        for (int32_t q = c.tail_lo + wid; q < c.tail_hi; q += NW) {
            const int32_t x = A.order[q];
            for (int64_t e0 = A.uptr[x]; e0 < A.uptr[x + 1]; e0 += 32) {
                const int64_t e = e0 + lane;
                bool hit = false;
                int32_t z = 0;
                if (e < A.uptr[x + 1]) {
                    z = A.unbr[e];
                    hit = moving[z] && A.comm[z] != frm;
                }
                const unsigned hm = __ballot_sync(0xffffffffu, hit);
                if (!hm) continue;
                unsigned long long at = 0;
                if (lane == 0) at = atomicAdd(&s_tot, (unsigned long long)__popc(hm));
                at = __shfl_sync(0xffffffffu, at, 0);
                if (fill && hit) {
                    const int64_t p = c.mv_off + (int64_t)at + __popc(hm & ((1u << lane) - 1));
                    mv_z[p] = z;
                    mv_u[p] = A.uu[e];
                    mv_e[p] = e;
                    mv_i[p] = (x == i);
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (fill) spec[k].mv_cnt = (int32_t)s_tot;
            else cnt[k] = (int64_t)s_tot;
        }
        __syncthreads();
    }
}

// ---- big candidates on integer-weight graphs, cut into work items of BIG_CH entries so that
// a coarse-level hub candidate (rows of ~10^6 entries) is spread over the whole GPU instead
// of one CTA.  Items: chunks of the tail members' rows (x >= 0) and of row i itself (x < 0,
// the attach target).  Tail sums are accumulated with fp64 atomics -- exact, since every
// partial sum is an integer below 2^53 -- and the attach target is reduced from per-item
// (gain, entry) partials with the reference's first-maximum rule.
constexpr int64_t BIG_CH = 4096;
struct BigItem {
    int32_t b, x;
    int64_t e0, e1;
};
__global__ void __launch_bounds__(256) k_big_count(CommitArgs A, const int32_t *big,
                                                   const int32_t *nbig, int64_t *cnt) {
    __shared__ unsigned long long s_c;
    const int32_t nb = *nbig;
    for (int32_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const int32_t k = big[b];
        const int32_t i = A.cand[k], frm = A.comm[i];
        int32_t lo, hi;
        tail_range(A, i, frm, lo, hi);
        if (threadIdx.x == 0) s_c = 0;
        __syncthreads();
        unsigned long long c = 0;
        for (int32_t q = lo + threadIdx.x; q < hi; q += blockDim.x) {
            const int32_t x = A.order[q];
            c += (unsigned long long)((A.uptr[x + 1] - A.uptr[x] + BIG_CH - 1) / BIG_CH);
        }
        if (threadIdx.x == 0) c += (unsigned long long)((A.uptr[i + 1] - A.uptr[i] + BIG_CH - 1) / BIG_CH);
        atomicAdd(&s_c, c);
        __syncthreads();
        if (threadIdx.x == 0) cnt[b] = (int64_t)s_c;
        __syncthreads();
    }
}
__global__ void __launch_bounds__(256) k_big_fill(CommitArgs A, const int32_t *big,
                                                  const int32_t *nbig, const int64_t *off,
                                                  BigItem *items, int64_t *ri_off, int32_t *ri_cnt) {
    __shared__ unsigned long long s_pos;
    const int32_t nb = *nbig;
    for (int32_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const int32_t k = big[b];
        const int32_t i = A.cand[k], frm = A.comm[i];
        int32_t lo, hi;
        tail_range(A, i, frm, lo, hi);
        if (threadIdx.x == 0) {
            // row i's chunks first (a contiguous range: the attach partials of b)
            const int64_t e0 = A.uptr[i], e1 = A.uptr[i + 1];
            int32_t t = 0;
            for (int64_t e = e0; e < e1; e += BIG_CH, t++)
                items[off[b] + t] = BigItem{b, -1, e, min(e1, e + BIG_CH)};
            ri_off[b] = off[b];
            ri_cnt[b] = t;
            s_pos = (unsigned long long)(off[b] + t);
        }
        __syncthreads();
        for (int32_t q = lo + threadIdx.x; q < hi; q += blockDim.x) {
            const int32_t x = A.order[q];
            const int64_t e0 = A.uptr[x], e1 = A.uptr[x + 1];
            const int64_t nch = (e1 - e0 + BIG_CH - 1) / BIG_CH;
            if (!nch) continue;
            const int64_t p = (int64_t)atomicAdd(&s_pos, (unsigned long long)nch);
            for (int64_t t = 0; t < nch; t++)
                items[p + t] = BigItem{b, x, e0 + t * BIG_CH, min(e1, e0 + (t + 1) * BIG_CH)};
        }
        __syncthreads();
    }
}
// one warp per item: tail chunks accumulate w_to / w_from, row-i chunks give attach partials
__global__ void k_big_items_spec(CommitArgs A, const int32_t *big, const BigItem *items,
                                 int64_t nit, double *acc_wt, double *acc_wf, double *part_bt,
                                 int64_t *part_be) {
    const int lane = threadIdx.x & 31;
    for (int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; it < nit;
         it += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const BigItem I = items[it];
        const int32_t k = big[I.b];
        const int32_t i = A.cand[k], frm = A.comm[i], to = A.cstar[i];
        if (I.x >= 0) {
            int32_t lo, hi;
            tail_range(A, i, frm, lo, hi);
            const int32_t base = A.cptr[frm], plo = lo - base, phi = hi - base;
            double wt = 0.0, wf = 0.0;
            for (int64_t e = I.e0 + lane; e < I.e1; e += 32) {
                const int32_t z = A.unbr[e];
                const int32_t cz = A.comm[z];
                if (cz == to) wt += A.uu[e];
                if (cz != frm) continue;
                const int32_t pz = A.pos[z];
                if (pz >= plo && pz < phi) continue;   // z inside the moved tail
                wf += A.uu[e];
            }
            wt = warp_sum(wt);
            wf = warp_sum(wf);
            if (lane == 0) {
                if (wt != 0.0) atomicAdd(acc_wt + I.b, wt);
                if (wf != 0.0) atomicAdd(acc_wf + I.b, wf);
            }
        } else {
            const double soi = A.s_out[i], sii = A.s_in[i];
            double bt = -INFINITY;
            int64_t be = INT64_MAX;
            for (int64_t e = I.e0 + lane; e < I.e1; e += 32) {
                const int32_t z = A.unbr[e];
                if (A.comm[z] != to) continue;
                const double pg = A.uu[e] / A.m - (soi * A.s_in[z] + sii * A.s_out[z]) / A.m2;
                if (pg > bt) {
                    bt = pg;
                    be = e;
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ot = __shfl_xor_sync(0xffffffffu, bt, off);
                const int64_t oe = __shfl_xor_sync(0xffffffffu, be, off);
                if (ot > bt || (ot == bt && oe < be)) {
                    bt = ot;
                    be = oe;
                }
            }
            if (lane == 0) {
                part_bt[it] = bt;
                part_be[it] = be;
            }
        }
    }
}
// one CTA per big candidate: tail strengths and volume, the item sums, the attach partials
__global__ void __launch_bounds__(256) k_big_finish(CommitArgs A, const int32_t *big,
                                                    const int32_t *nbig, const double *acc_wt,
                                                    const double *acc_wf, const double *part_bt,
                                                    const int64_t *part_be, const int64_t *ri_off,
                                                    const int32_t *ri_cnt, CandSpec *spec,
                                                    int64_t *vol_out) {
    __shared__ double s_so[8], s_si[8];
    __shared__ unsigned long long s_vol;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int32_t nb = *nbig;
    for (int32_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const int32_t k = big[b];
        const int32_t i = A.cand[k], frm = A.comm[i];
        int32_t lo, hi;
        tail_range(A, i, frm, lo, hi);
        if (threadIdx.x == 0) s_vol = 0;
        __syncthreads();
        double so = 0.0, si = 0.0;
        unsigned long long vol = 0;
        for (int32_t q = lo + threadIdx.x; q < hi; q += blockDim.x) {
            const int32_t x = A.order[q];
            so += A.s_out[x];
            si += A.s_in[x];
            vol += (unsigned long long)(A.uptr[x + 1] - A.uptr[x]);
        }
        so = warp_sum(so);
        si = warp_sum(si);
        atomicAdd(&s_vol, vol);
        if (lane == 0) {
            s_so[wid] = so;
            s_si[wid] = si;
        }
        __syncthreads();
        if (wid == 0) {
            so = warp_sum(lane < 8 ? s_so[lane] : 0.0);
            si = warp_sum(lane < 8 ? s_si[lane] : 0.0);
            double bt = -INFINITY;
            int64_t be = INT64_MAX;
            for (int32_t t = lane; t < ri_cnt[b]; t += 32) {
                const double ot = part_bt[ri_off[b] + t];
                const int64_t oe = part_be[ri_off[b] + t];
                if (ot > bt || (ot == bt && oe < be)) {
                    bt = ot;
                    be = oe;
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ot = __shfl_xor_sync(0xffffffffu, bt, off);
                const int64_t oe = __shfl_xor_sync(0xffffffffu, be, off);
                if (ot > bt || (ot == bt && oe < be)) {
                    bt = ot;
                    be = oe;
                }
            }
            if (lane == 0) {
                vol_out[k] = (int64_t)s_vol;
                CandSpec c;
                c.w_to = acc_wt[b];
                c.w_from = acc_wf[b];
                c.so_b = so;
                c.si_b = si;
                c.pgj = bt;
                c.je = be != INT64_MAX ? be : -1;
                c.mv_off = 0;
                c.j = be != INT64_MAX ? A.unbr[be] : -1;
                c.tail_lo = lo;
                c.tail_hi = hi;
                c.mv_cnt = -1;   // big: k_mv_scan leaves it to the big moving-neighbour scan
                spec[k] = c;
            }
        }
        __syncthreads();
    }
}
// moving-neighbour entries of the big candidates' tail items (any order: re-pricing breaks ties
// by entry index); per-candidate positions from a counter, mv_cnt set by k_big_mv_finish
__global__ void k_big_items_mv(CommitArgs A, const int32_t *big, const BigItem *items, int64_t nit,
                               const CandSpec *spec, const uint8_t *moving,
                               unsigned long long *ctr, int32_t *mv_z, double *mv_u, int64_t *mv_e,
                               uint8_t *mv_i) {
    const int lane = threadIdx.x & 31;
    for (int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; it < nit;
         it += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const BigItem I = items[it];
        if (I.x < 0) continue;
        const int32_t k = big[I.b];
        const int32_t i = A.cand[k], frm = A.comm[i];
        const int64_t mo = spec[k].mv_off;
        for (int64_t e0 = I.e0; e0 < I.e1; e0 += 32) {
            const int64_t e = e0 + lane;
            bool hit = false;
            int32_t z = 0;
            if (e < I.e1) {
                z = A.unbr[e];
                hit = moving[z] && A.comm[z] != frm;
            }
            const unsigned hm = __ballot_sync(0xffffffffu, hit);
            if (!hm) continue;
            unsigned long long at = 0;
            if (lane == 0) at = atomicAdd(ctr + I.b, (unsigned long long)__popc(hm));
            at = __shfl_sync(0xffffffffu, at, 0);
            if (hit) {
                const int64_t p = mo + (int64_t)at + __popc(hm & ((1u << lane) - 1));
                mv_z[p] = z;
                mv_u[p] = A.uu[e];
                mv_e[p] = e;
                mv_i[p] = (I.x == i);
            }
        }
    }
}
__global__ void k_big_mv_finish(const int32_t *big, const int32_t *nbig,
                                const unsigned long long *ctr, CandSpec *spec) {
    GS_LOOP(b, *nbig) spec[big[b]].mv_cnt = (int32_t)ctr[b];
}

__global__ void k_mv_offsets(int64_t K, const int32_t *status, const int64_t *off, CandSpec *spec) {
    GS_LOOP(k, K) if (status[k] == ST_UNRES) spec[k].mv_off = off[k];
}

struct MvList {
    const int32_t *z;
    const double *u;
    const int64_t *e;
    const uint8_t *is_i;
};

// exact re-pricing of candidate (i -> C) against the live labels: w_to and the attach target
__device__ void reprice(const CommitArgs &A, const MvList &M, const int32_t *lab, const CandSpec &c,
                        int32_t i, int32_t C, double &wt, int32_t &j) {
    const int lane = threadIdx.x & 31;
    double dw = 0.0;
    double bt = -INFINITY;
    int64_t be = INT64_MAX;
    int lost = 0;
    const double soi = A.s_out[i], sii = A.s_in[i];
    for (int32_t t = lane; t < c.mv_cnt; t += 32) {
        const int64_t q = c.mv_off + t;
        const int32_t z = M.z[q];
        const bool now = lab[z] == C, was = A.comm[z] == C;
        if (now != was) dw += now ? M.u[q] : -M.u[q];
        if (M.is_i[q]) {
            if (now) {
                const double pg = M.u[q] / A.m - (soi * A.s_in[z] + sii * A.s_out[z]) / A.m2;
                const int64_t e = M.e[q];
                if (pg > bt || (pg == bt && e < be)) {
                    bt = pg;
                    be = e;
                }
            } else if (was && z == c.j) {
                lost = 1;
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        dw += __shfl_xor_sync(0xffffffffu, dw, off);
        lost |= __shfl_xor_sync(0xffffffffu, lost, off);
        const double ot = __shfl_xor_sync(0xffffffffu, bt, off);
        const int64_t oe = __shfl_xor_sync(0xffffffffu, be, off);
        if (ot > bt || (ot == bt && oe < be)) {
            bt = ot;
            be = oe;
        }
    }
    wt = c.w_to + dw;
    if (lost) {   // the snapshot attach target itself left C: rescan i's row
        attach_only(A.uptr, A.unbr, A.uu, A.s_out, A.s_in, lab, i, C, A.m, A.m2, j);
        return;
    }
    j = c.j;
    if (be != INT64_MAX && (c.j < 0 || bt > c.pgj || (bt == c.pgj && be < c.je))) j = A.unbr[be];
}

__global__ void k_acc_flags(int64_t K, const int32_t *status, int32_t *f) {
    GS_LOOP(k, K) f[k] = status[k] == ST_UNRES ? 1 : 0;
}
__global__ void k_acc_pairs(const int32_t *cand, const int32_t *comm, const int32_t *cstar,
                            int64_t K, const int32_t *f, const int32_t *pos, uint32_t *key,
                            int32_t *val) {
    GS_LOOP(k, K) {
        if (!f[k]) continue;
        const int32_t i = cand[k];
        const int64_t t = 2 * (int64_t)pos[k];
        key[t] = (uint32_t)comm[i];
        val[t] = (int32_t)k;
        key[t + 1] = (uint32_t)cstar[i];
        val[t + 1] = (int32_t)k;
    }
}
__global__ void k_lb32c(const uint32_t *sorted, int64_t m, int64_t nrows, int32_t *ptr) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= nrows;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = m;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if ((int64_t)sorted[mid] < r) lo = mid + 1;
            else hi = mid;
        }
        ptr[r] = (int32_t)lo;
    }
}
__global__ void k_ev_rec(const int32_t *ev, int64_t m, const int32_t *cand, const int32_t *comm,
                         const int32_t *cstar, int4 *rec) {
    GS_LOOP(q, m) {
        const int32_t k = ev[q], i = cand[k];
        rec[q] = make_int4(k, i, comm[i], cstar[i]);
    }
}
__global__ void k_walker_list(const int32_t *tl_ptr, int64_t nc, int32_t *f) {
    GS_LOOP(c, nc) f[c] = tl_ptr[c + 1] > tl_ptr[c] ? 1 : 0;
}
// walker list and initial walker state.  A walker whose first event moves a candidate out of
// its community starts parked at that event (atk = k): its state is the initial one, exactly
// what its first visit would publish, so the target's walker can evaluate the event at once
// instead of waiting for that visit (a hub community's timeline is mostly such events).
__global__ void k_walker_scatter(const int32_t *f, const int32_t *pos, const int32_t *tl_ptr,
                                 const int4 *tl_rec, int64_t nc, int32_t *wl, int32_t *wpos,
                                 int32_t *atk, int2 *wwait) {
    GS_LOOP(c, nc) {
        int32_t at = 0x7fffffff;
        if (f[c]) {
            wl[pos[c]] = (int32_t)c;
            const int4 r = tl_rec[tl_ptr[c]];
            if (r.w != (int32_t)c) {   // first event: c is its source
                at = r.x;
                wwait[c] = make_int2(r.x, -1);
            }
        }
        wpos[c] = tl_ptr[c];
        atk[c] = at;
    }
}

struct Live {
    int32_t *lab;
    double *S_out, *S_in;
    int32_t *cnt;
    uint8_t *dirty;
    int32_t *first_commit;
    int32_t *a;
    int32_t *wpos, *atk;
    int2 *wwait;             // per walker: what a parked walker waits for ({k, frm} or {-1, -1})
    const int32_t *tl_ptr, *tl_ev;
    const int4 *tl_rec;      // per timeline event: {k, i, frm, to}
    MvList mv;
    double *gain;
    int32_t *remaining;
    unsigned long long *wst;   // SLM_PROFILE_WALK counters (else nullptr)
};

__device__ __forceinline__ int32_t vload(const int32_t *p) { return *(volatile const int32_t *)p; }
// acquire load (gpu scope): later loads are not performed before it, and writes released by a
// fence + store on another SM are visible after it -- unlike __threadfence(), it does not wait
// for this thread's own earlier stores to drain
__device__ __forceinline__ int32_t ld_acq(const int32_t *p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// resolve an accepted candidate as skipped exactly once (both of its walkers may try)
__device__ __forceinline__ void resolve_skip(int32_t *status, int32_t k, int32_t *remaining) {
    if (atomicCAS(status + k, ST_UNRES, ST_SKIP) == ST_UNRES) atomicSub(remaining, 1);
}
__device__ __forceinline__ uint8_t vload8(const uint8_t *p) { return *(volatile const uint8_t *)p; }

// per-lane exact re-pricing (serial over the candidate's moving-neighbour entries); false
// when the snapshot attach target left C (the row must be rescanned cooperatively)
__device__ bool reprice_lane(const CommitArgs &A, const MvList &M, const int32_t *lab,
                             const CandSpec &c, int32_t i, int32_t C, double &wt, int32_t &j) {
    double dw = 0.0, bt = -INFINITY;
    int64_t be = INT64_MAX;
    bool lost = false;
    const double soi = A.s_out[i], sii = A.s_in[i];
    for (int32_t t = 0; t < c.mv_cnt; t++) {
        const int64_t q = c.mv_off + t;
        const int32_t z = M.z[q];
        const bool now = lab[z] == C, was = A.comm[z] == C;
        if (now != was) dw += now ? M.u[q] : -M.u[q];
        if (M.is_i[q]) {
            if (now) {
                const double pg = M.u[q] / A.m - (soi * A.s_in[z] + sii * A.s_out[z]) / A.m2;
                const int64_t e = M.e[q];
                if (pg > bt || (pg == bt && e < be)) {
                    bt = pg;
                    be = e;
                }
            } else if (was && z == c.j) {
                lost = true;
            }
        }
    }
    wt = c.w_to + dw;
    if (lost) return false;
    j = c.j;
    if (be != INT64_MAX && (c.j < 0 || bt > c.pgj || (bt == c.pgj && be < c.je))) j = A.unbr[be];
    return true;
}

// A walker walks one community's timeline (see header comment).  Up to 32 upcoming events
// are loaded by the lanes of a warp and classified in parallel against C's current state
// (speculation: every event up to the first state-changing one -- a commit into C, an
// observed commit out of C, or a wait -- sees exactly that state); skips before it are
// written at once, the barrier event is applied, and the rest of the batch is reclassified.
// A candidate's status is written only by its target's walker (the source side merely
// moves past a certain skip), so resolutions need no CAS and `remaining` drops once per
// walker visit.  Long timelines (hub communities: ~10^5 events, a few dozen commits) are
// walked by a whole CTA: its threads classify 256 events at a time and write the skips
// before the first state-changing event, and warp 0 applies that event with the warp logic.
enum { C_PASS = 0, C_SKIP = 1, C_COMMIT = 2, C_OUTCOMMIT = 3, C_WAIT = 4, C_COOP = 5 };

struct WalkState {
    double SoC, SiC;
    int32_t cntC, my_atk;
    int dirtyC;
    int win;   // classification window: events classified per round (adapts to barrier density)
};

// one event as a lane sees it
struct WalkEv {
    int32_t k, i, frm, to, atF, st;
    int dF;
    double SoF, SiF;
    CandSpec cs;
};
__device__ __forceinline__ void walk_load(const Live &V, const int32_t *status, const CandSpec *spec,
                                          int32_t C, bool valid, int4 rec, WalkEv &e) {
    e.k = -1;
    e.i = 0;
    e.frm = 0;
    e.to = -1;
    e.atF = -1;
    e.st = ST_SKIP;
    e.dF = 0;
    e.SoF = e.SiF = 0.0;
    e.cs.w_to = e.cs.w_from = e.cs.so_b = e.cs.si_b = e.cs.pgj = 0.0;
    e.cs.je = -1;
    e.cs.mv_off = 0;
    e.cs.j = -1;
    e.cs.tail_lo = e.cs.tail_hi = 0;
    e.cs.mv_cnt = 0;
    if (valid) {
        e.k = rec.x;
        e.i = rec.y;
        e.frm = rec.z;
        e.to = rec.w;
        e.st = ld_acq(status + e.k);
        if (e.to == C && e.st == ST_UNRES) {
            e.atF = ld_acq(V.atk + e.frm);
            e.dF = vload8(V.dirty + e.frm);
            e.SoF = V.S_out[e.frm];
            e.SiF = V.S_in[e.frm];
            e.cs = spec[e.k];
        }
    }
}

// classification of one event against C's state W (lane-local; may refresh e's source state)
__device__ __forceinline__ int walk_classify(const CommitArgs &A, const Live &V, int32_t *status,
                                             int32_t C, const WalkState &W, WalkEv &e, double &gq,
                                             double &wtq, int32_t &jq) {
    int cls = C_PASS;
    gq = 0.0;
    wtq = 0.0;
    jq = -1;
    const int32_t k = e.k, frm = e.frm;
    if (e.to != C) {   // C is the source
        if (e.st == ST_COMMIT) {
            cls = C_OUTCOMMIT;
        } else if (e.st == ST_UNRES && !(W.my_atk != k && W.dirtyC)) {
            e.st = ld_acq(status + k);
            cls = e.st == ST_COMMIT ? C_OUTCOMMIT : (e.st == ST_UNRES ? C_WAIT : C_PASS);
        }
    } else if (e.st == ST_UNRES) {   // C evaluates k
        int undecided = 1;
        if (W.cntC == 0 || e.dF) {
            cls = C_SKIP;
            undecided = 0;
        } else if (e.atF != k) {
            e.atF = ld_acq(V.atk + frm);
            if (e.atF != k) {
                cls = vload8(V.dirty + frm) ? C_SKIP : C_WAIT;
                if (cls == C_SKIP) e.dF = 1;
                undecided = 0;
            } else {
                if (vload8(V.dirty + frm)) {
                    e.dF = 1;
                    cls = C_SKIP;
                    undecided = 0;
                } else {
                    e.SoF = V.S_out[frm];
                    e.SiF = V.S_in[frm];
                }
            }
        }
        if (undecided) {
            const CandSpec &cs = e.cs;
            wtq = cs.w_to;
            jq = cs.j;
            // long list, lost attach target, or a dense stretch of commits (small window: the
            // event is priced by the whole warp rather than one lane): cooperative
            if (cs.mv_cnt > 0 && W.dirtyC &&
                (cs.mv_cnt > 64 || W.win <= 4 || !reprice_lane(A, V.mv, V.lab, cs, e.i, C, wtq, jq))) {
                cls = C_COOP;
            } else {
                const double so_b = cs.so_b, si_b = cs.si_b;
                // gain_switch d_null (quality.py:216-219), exact operand order
                const double d_null = -e.SoF * si_b - so_b * e.SiF + W.SoC * si_b +
                                      so_b * W.SiC + 2.0 * so_b * si_b;
                gq = (wtq - cs.w_from) / A.m - d_null / (A.m * A.m);
                cls = (gq > 0.0 && jq >= 0) ? C_COMMIT : C_SKIP;   // detector.py:498-502
            }
        }
    }
    return cls;
}

// after a commit into C, the batch's following events [s0, nb) are decided in one pass while
// they stay simple: candidates into C with a parked clean source and no moving neighbour
// (their w_to is the snapshot's, whatever moved) and resolved skips out of C.  The
// decisions are the serial ones: the lanes replay them in order with C's running totals (a
// commit also marks later candidates out of the same source), then apply every commit's
// state at once, fence, and publish the verdicts.  Returns the first event left undecided.
__device__ __forceinline__ int walk_run(const CommitArgs &A, const Live &V, int32_t *status,
                                        int32_t C, int s0, int nb, WalkEv &e, WalkState &W,
                                        int &nres, int &ncommit) {
    const int lane = threadIdx.x & 31;
    // 0 stop, 1 no effect, 2 skip, 3 gain decides
    int kind = 1;
    if (lane >= s0 && lane < nb) {
        if (e.to != C) {
            kind = e.st == ST_SKIP ? 1 : 0;
        } else if (e.st != ST_UNRES) {
            kind = 1;
        } else if (e.dF) {
            kind = 2;
        } else {
            if (e.atF != e.k) {
                e.atF = ld_acq(V.atk + e.frm);
                if (e.atF == e.k) {
                    e.SoF = V.S_out[e.frm];
                    e.SiF = V.S_in[e.frm];
                }
            }
            const int df = vload8(V.dirty + e.frm);
            if (df) kind = 2;
            else if (e.atF != e.k) kind = 0;
            else kind = e.cs.mv_cnt > 0 ? 4 : 3;
        }
    }
    int end = nb;
    int mydec = 0;   // 1 skip, 2 commit
    double myg = 0.0;
    for (int l = s0; l < nb; l++) {
        const int kl = __shfl_sync(0xffffffffu, kind, l);
        if (kl <= 0) {
            end = l;
            if (V.wst && lane == 0) atomicAdd(V.wst + (kl < 0 ? 3 : 4), 1ull);
            break;
        }
        if (kl == 1) continue;
        const int dl = __shfl_sync(0xffffffffu, e.dF, l);
        const double so_b = __shfl_sync(0xffffffffu, e.cs.so_b, l);
        const double si_b = __shfl_sync(0xffffffffu, e.cs.si_b, l);
        const double SoF = __shfl_sync(0xffffffffu, e.SoF, l);
        const double SiF = __shfl_sync(0xffffffffu, e.SiF, l);
        double wt = __shfl_sync(0xffffffffu, e.cs.w_to, l);
        const double wf = __shfl_sync(0xffffffffu, e.cs.w_from, l);
        int32_t jl = __shfl_sync(0xffffffffu, e.cs.j, l);
        if (kl == 4 && !dl) {
            // moving neighbours: the whole warp re-prices the candidate now, the labels of
            // every commit before it (this run's included) being written
            CandSpec c;
            c.w_to = wt;
            c.w_from = wf;
            c.so_b = so_b;
            c.si_b = si_b;
            c.j = jl;
            c.tail_lo = __shfl_sync(0xffffffffu, e.cs.tail_lo, l);
            c.tail_hi = __shfl_sync(0xffffffffu, e.cs.tail_hi, l);
            c.pgj = __shfl_sync(0xffffffffu, e.cs.pgj, l);
            c.je = __shfl_sync(0xffffffffu, e.cs.je, l);
            c.mv_off = __shfl_sync(0xffffffffu, e.cs.mv_off, l);
            c.mv_cnt = __shfl_sync(0xffffffffu, e.cs.mv_cnt, l);
            const int32_t il = __shfl_sync(0xffffffffu, e.i, l);
            reprice(A, V.mv, V.lab, c, il, C, wt, jl);
        }
        const int32_t fl = __shfl_sync(0xffffffffu, e.frm, l);
        const int32_t len = __shfl_sync(0xffffffffu, e.cs.tail_hi - e.cs.tail_lo, l);
        bool commit = false;
        double g = 0.0;
        if (kl >= 3 && !dl) {
            // gain_switch d_null (quality.py:216-219), exact operand order
            const double d_null = -SoF * si_b - so_b * SiF + W.SoC * si_b + so_b * W.SiC +
                                  2.0 * so_b * si_b;
            g = (wt - wf) / A.m - d_null / (A.m * A.m);
            commit = g > 0.0 && jl >= 0;   // detector.py:498-502
        }
        if (lane == l) {
            mydec = commit ? 2 : 1;
            myg = g;
            if (commit) {
                for (int32_t t = e.cs.tail_lo; t < e.cs.tail_hi; t++) V.lab[A.order[t]] = C;
                e.cs.j = jl;
            }
        }
        if (commit) {
            __syncwarp();   // the labels before any later re-pricing
            W.SoC += so_b;
            W.SiC += si_b;
            W.cntC += len;
            if (lane > l && e.frm == fl) e.dF = 1;   // later candidates out of the same source
        }
    }
    const unsigned cm = __ballot_sync(0xffffffffu, mydec == 2);
    if (mydec == 2) {
        const int32_t len = e.cs.tail_hi - e.cs.tail_lo;
        V.a[e.i] = e.cs.j;   // (the re-priced attach target)
        // move_nodes (quality.py:87-95)
        V.S_out[e.frm] -= e.cs.so_b;
        V.S_in[e.frm] -= e.cs.si_b;
        V.cnt[e.frm] -= len;
        V.dirty[e.frm] = 1;
        atomicMin(&V.first_commit[e.frm], e.k);
        atomicMin(&V.first_commit[C], e.k);
        V.gain[e.k] = myg;
    }
    if (cm && lane == 0) {
        V.S_out[C] = W.SoC;
        V.S_in[C] = W.SiC;
        V.cnt[C] = W.cntC;
        V.dirty[C] = 1;
    }
    __syncwarp();
    if (cm) __threadfence();   // state and labels before the verdicts
    __syncwarp();
    if (mydec) {
        *(volatile int32_t *)(status + e.k) = mydec == 2 ? ST_COMMIT : ST_SKIP;
        e.st = mydec == 2 ? ST_COMMIT : ST_SKIP;
    }
    nres += __popc(__ballot_sync(0xffffffffu, mydec != 0));
    ncommit += __popc(cm);
    return end;
}

// one warp batch: the events [p, p + nb) (lane < nb holds event p + lane, record rec) against
// W; returns the events consumed (nb, or fewer when the walker parks)
__device__ __forceinline__ int walk_batch(const CommitArgs &A, const Live &V, int32_t *status,
                          const CandSpec *spec, int32_t C, int4 rec, int nb, WalkState &W,
                          int &nres, bool &parked, int &ncommit, int &nbarrier, int &nchg) {
    const int lane = threadIdx.x & 31;
    WalkEv e;
    walk_load(V, status, spec, C, lane < nb, rec, e);
    int start = 0;
    while (start < nb) {
        // ---- classify events [start, hi) against the current state.  Every event after a
        // state change is classified again, so dense stretches of commits (a hub community
        // absorbing most of a sweep's candidates) shrink the window instead of re-pricing the
        // whole batch after each commit
        const int hi = min(nb, start + W.win);
        const bool act = lane >= start && lane < hi;
        int cls = C_PASS;
        double gq = 0.0, wtq = 0.0;
        int32_t jq = -1;
        if (act) cls = walk_classify(A, V, status, C, W, e, gq, wtq, jq);
        // ---- skips before the first state-changing event
        const unsigned bar = __ballot_sync(0xffffffffu, act && cls >= C_COMMIT);
        const int f = bar ? __ffs(bar) - 1 : hi;
        const bool sk = act && lane < f && cls == C_SKIP;
        if (sk) *(volatile int32_t *)(status + e.k) = ST_SKIP;
        nres += __popc(__ballot_sync(0xffffffffu, sk));
        if (f >= hi) {   // no state change in the window
            W.win = min(32, W.win * 2);
            start = hi;
            continue;
        }
        W.win = (f - start) * 4 < W.win ? max(1, W.win >> 1) : min(32, W.win * 2);
        const int cf = __shfl_sync(0xffffffffu, cls, f);
        const int32_t kf = __shfl_sync(0xffffffffu, e.k, f);
        if (cf == C_WAIT) {
            // what unblocks it: the verdict on kf (C is its source), or kf's source walker
            // parking at kf / turning dirty (C is its target)
            const int32_t tf = __shfl_sync(0xffffffffu, e.to, f);
            const int32_t ff = __shfl_sync(0xffffffffu, e.frm, f);
            if (lane == 0) {
                if (W.my_atk != kf) {
                    __threadfence();
                    *(volatile int32_t *)(V.atk + C) = kf;
                }
                V.wwait[C] = make_int2(kf, tf == C ? ff : -1);
            }
            W.my_atk = kf;
            parked = true;
            return f;
        }
        nchg++;
        if (cf == C_OUTCOMMIT) {   // our state was changed by that commit (its status was
                                   // read with acquire: the state is visible)
            W.SoC = V.S_out[C];
            W.SiC = V.S_in[C];
            W.cntC = V.cnt[C];
            W.dirtyC = 1;
            start = f + 1;
            continue;
        }
        // ---- evaluated candidate kf into C (commit, or a cooperative re-pricing)
        const int32_t iq = __shfl_sync(0xffffffffu, e.i, f);
        const int32_t fq = __shfl_sync(0xffffffffu, e.frm, f);
        const double so_b = __shfl_sync(0xffffffffu, e.cs.so_b, f);
        const double si_b = __shfl_sync(0xffffffffu, e.cs.si_b, f);
        const int32_t tlo = __shfl_sync(0xffffffffu, e.cs.tail_lo, f);
        const int32_t thi = __shfl_sync(0xffffffffu, e.cs.tail_hi, f);
        double g = __shfl_sync(0xffffffffu, gq, f);
        int32_t j = __shfl_sync(0xffffffffu, jq, f);
        bool commit = cf == C_COMMIT;
        if (cf == C_COOP) {
            CandSpec c;
            c.w_to = __shfl_sync(0xffffffffu, e.cs.w_to, f);
            c.w_from = __shfl_sync(0xffffffffu, e.cs.w_from, f);
            c.so_b = so_b;
            c.si_b = si_b;
            c.j = __shfl_sync(0xffffffffu, e.cs.j, f);
            c.tail_lo = tlo;
            c.tail_hi = thi;
            c.pgj = __shfl_sync(0xffffffffu, e.cs.pgj, f);
            c.je = __shfl_sync(0xffffffffu, e.cs.je, f);
            c.mv_off = __shfl_sync(0xffffffffu, e.cs.mv_off, f);
            c.mv_cnt = __shfl_sync(0xffffffffu, e.cs.mv_cnt, f);
            const double SoFq = __shfl_sync(0xffffffffu, e.SoF, f);
            const double SiFq = __shfl_sync(0xffffffffu, e.SiF, f);
            double wt = c.w_to;
            reprice(A, V.mv, V.lab, c, iq, C, wt, j);
            const double d_null = -SoFq * si_b - so_b * SiFq + W.SoC * si_b + so_b * W.SiC +
                                  2.0 * so_b * si_b;
            g = (wt - c.w_from) / A.m - d_null / (A.m * A.m);
            commit = g > 0.0 && j >= 0;
        }
        nbarrier++;
        if (commit) {
            ncommit++;
            const int32_t len = thi - tlo;
            if (V.wst && lane == 0) atomicAdd(V.wst + 5, (unsigned long long)len);
            for (int32_t t = tlo + lane; t < thi; t += 32) V.lab[A.order[t]] = C;
            W.SoC += so_b;
            W.SiC += si_b;
            W.cntC += len;
            W.dirtyC = 1;
            if (e.frm == fq) e.dF = 1;   // later candidates out of the same source skip
            if (lane == 0) {
                V.a[iq] = j;
                // move_nodes (quality.py:87-95)
                V.S_out[fq] -= so_b;
                V.S_in[fq] -= si_b;
                V.cnt[fq] -= len;
                V.S_out[C] = W.SoC;
                V.S_in[C] = W.SiC;
                V.cnt[C] = W.cntC;
                V.dirty[fq] = 1;
                V.dirty[C] = 1;
                atomicMin(&V.first_commit[fq], kf);
                atomicMin(&V.first_commit[C], kf);
                V.gain[kf] = g;
            }
        }
        __syncwarp();
        if (lane == 0) {
            if (commit) __threadfence();   // state and labels before the verdict
            *(volatile int32_t *)(status + kf) = commit ? ST_COMMIT : ST_SKIP;
        }
        if (lane == f) e.st = commit ? ST_COMMIT : ST_SKIP;
        nres++;
        start = f + 1;
        if (commit && A.runs && start < nb)
            start = walk_run(A, V, status, C, start, nb, e, W, nres, ncommit);
    }
    return nb;
}

__device__ __forceinline__ void walk_state_load(const Live &V, int32_t C, WalkState &W) {
    W.SoC = V.S_out[C];
    W.SiC = V.S_in[C];
    W.cntC = V.cnt[C];
    W.my_atk = V.atk[C];             // only this walker writes atk[C]
    W.dirtyC = vload8(V.dirty + C);  // monotone
    W.win = 32;
}

// end of a visit: resolved count, position, and release of waiters when the timeline is done
__device__ __forceinline__ void walk_visit_end(const Live &V, int32_t C, int32_t p, int32_t end,
                                               int nres) {
    if (nres) atomicSub(V.remaining, nres);
    V.wpos[C] = p;
    if (p >= end) {
        __threadfence();
        *(volatile int32_t *)(V.atk + C) = 0x7fffffff;
    }
}

constexpr int WALK_BLOCK = 256;
constexpr int WALK_CLEAN = 4;   // clean warp batches before a CTA walker resumes scanning

// persistent walkers: blocks [0, nlong) walk the long timelines wlong[b] with the whole CTA;
// the warps of the other blocks walk wl (skipping the CTA-walked communities).  The grid is
// resident, so a parked walker resumes as soon as its verdict is written.
__global__ void __launch_bounds__(WALK_BLOCK) k_walk(CommitArgs A, Live V, const int32_t *wl,
                                                     int64_t nw_, int32_t *status,
                                                     const CandSpec *spec, int persistent,
                                                     const int32_t *wlong, int32_t nlong,
                                                     const uint8_t *cta_mode) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if ((int32_t)blockIdx.x < nlong) {
        // ---------------------------------------------------------------- CTA walker
        __shared__ int s_f, s_cnt, s_parked, s_p;
        __shared__ WalkState s_W;
        const int32_t C = wlong[blockIdx.x];
        const int32_t end = V.tl_ptr[C + 1];
        for (;;) {
            int32_t p = V.wpos[C];
            if (p >= end) break;
            __threadfence();
            WalkState W;
            walk_state_load(V, C, W);
            const int32_t p_start = p;
            int nres = 0;   // (thread 0's count)
            bool parked = false;
            int ncommit = 0, nbarrier = 0;
            while (p < end && !parked) {
                // skip scan: WALK_BLOCK events against the current state
                const int nbk = min(WALK_BLOCK, end - p);
                const int t = threadIdx.x;
                if (t == 0) {
                    s_f = nbk;
                    s_cnt = 0;
                }
                __syncthreads();
                WalkEv e;
                const bool valid = t < nbk;
                walk_load(V, status, spec, C, valid, valid ? V.tl_rec[p + t] : make_int4(-1, 0, 0, -1), e);
                int cls = C_PASS;
                double gq, wtq;
                int32_t jq;
                if (valid) cls = walk_classify(A, V, status, C, W, e, gq, wtq, jq);
                if (valid && cls >= C_COMMIT) atomicMin(&s_f, t);
                __syncthreads();
                const int f = s_f;
                const bool sk = valid && t < f && cls == C_SKIP;
                if (sk) *(volatile int32_t *)(status + e.k) = ST_SKIP;
                const int ns = __popc(__ballot_sync(0xffffffffu, sk));
                if (lane == 0 && ns) atomicAdd(&s_cnt, ns);
                __syncthreads();
                if (t == 0) nres += s_cnt;
                p += f;
                if (f >= nbk) continue;   // no state change in this window
                // the state-changing event at p: warp 0 applies it with the warp logic and
                // keeps walking by warp batches while state changes are dense (early sweeps);
                // WALK_CLEAN consecutive batches without one return to the CTA scan
                if (wid == 0) {
                    int nr = 0;
                    bool pk = false;
                    int32_t q = p;
                    int clean = 0;
                    int4 rec_next = lane < min(32, end - q) ? V.tl_rec[q + lane]
                                                            : make_int4(-1, 0, 0, -1);
                    while (q < end) {
                        const int nb = min(32, end - q);
                        const int4 rec = rec_next;
                        rec_next = q + nb + lane < end ? V.tl_rec[q + nb + lane]
                                                       : make_int4(-1, 0, 0, -1);
                        int nchg = 0;
                        q += walk_batch(A, V, status, spec, C, rec, nb, W, nr, pk, ncommit,
                                        nbarrier, nchg);
                        if (pk) break;
                        clean = nchg ? 0 : clean + 1;
                        if (clean >= WALK_CLEAN) break;
                    }
                    if (lane == 0) {
                        s_W = W;
                        s_p = q;
                        s_parked = pk ? 1 : 0;
                        nres += nr;
                    }
                }
                __syncthreads();
                W = s_W;
                p = s_p;
                parked = s_parked != 0;
                __syncthreads();
            }
            if (threadIdx.x == 0) {
                if (V.wst && p > p_start) {
                    atomicAdd(V.wst, (unsigned long long)(p - p_start));
                    atomicMax(V.wst + 1, (unsigned long long)(p - p_start));
                    atomicAdd(V.wst + 2, 1ull);
                    atomicMax(V.wst + 6, (unsigned long long)ncommit);
                    atomicMax(V.wst + 7, (unsigned long long)nbarrier);
                }
                walk_visit_end(V, C, p, end, nres);
            }
            __syncthreads();
            if (!persistent || p >= end) break;
            if (p == p_start) __nanosleep(256);
        }
        return;
    }
    // -------------------------------------------------------------------- warp walkers
    int64_t w = ((blockIdx.x - nlong) * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((gridDim.x - nlong) * (int64_t)blockDim.x) >> 5;
    for (;;) {
    int pending = 0, progressed = 0;
    for (int64_t wi = w; wi < nw_; wi += nwarps) {
        const int32_t C = wl[wi];
        if (cta_mode && cta_mode[C]) continue;
        int32_t p = V.wpos[C];
        const int32_t end = V.tl_ptr[C + 1];
        if (p >= end) continue;
        {   // a parked walker whose wait still holds is skipped without a visit
            const int2 ww = V.wwait[C];
            if (ww.x >= 0) {
                const bool blocked =
                    ww.y < 0 ? ld_acq(status + ww.x) == ST_UNRES
                             : (ld_acq(V.atk + ww.y) != ww.x && !vload8(V.dirty + ww.y));
                if (blocked) {
                    pending = 1;
                    continue;
                }
            }
        }
        __threadfence();
        WalkState W;
        walk_state_load(V, C, W);
        int nres = 0;                       // candidates resolved by this visit
        int ncommit = 0, nbarrier = 0;      // (profiling)
        bool parked = false;
        const int32_t p_start = p;
        // event records {k, i, frm, to} of the next batch are loaded one batch ahead
        int4 rec_next = make_int4(-1, 0, 0, -1);
        if (p + lane < end) rec_next = V.tl_rec[p + lane];
        while (p < end && !parked) {
            const int nb = min(32, end - p);
            const int4 rec = rec_next;
            rec_next = make_int4(-1, 0, 0, -1);
            if (p + nb + lane < end) rec_next = V.tl_rec[p + nb + lane];
            int nchg = 0;
            p += walk_batch(A, V, status, spec, C, rec, nb, W, nres, parked, ncommit, nbarrier, nchg);
        }
        if (V.wst && lane == 0 && p > p_start) {
            atomicAdd(V.wst, (unsigned long long)(p - p_start));
            atomicMax(V.wst + 1, (unsigned long long)(p - p_start));
            atomicAdd(V.wst + 2, 1ull);
            atomicMax(V.wst + 6, (unsigned long long)ncommit);
            atomicMax(V.wst + 7, (unsigned long long)nbarrier);
        }
        if (lane == 0) walk_visit_end(V, C, p, end, nres);
        if (p > p_start) progressed = 1;
        if (p < end) pending = 1;
    }
    if (!persistent || !pending) break;
    if (!progressed) __nanosleep(256);
    }
}

__global__ void k_long_flags(const int32_t *wl, int64_t nw, const int32_t *tl_ptr, int32_t lim,
                             int32_t *f) {
    GS_LOOP(q, nw) {
        const int32_t c = wl[q];
        f[q] = tl_ptr[c + 1] - tl_ptr[c] > lim ? 1 : 0;
    }
}
__global__ void k_long_scatter(const int32_t *f, const int32_t *pos, const int32_t *wl, int64_t nw,
                               int32_t nlong, int32_t *wlong, uint8_t *cmode) {
    GS_LOOP(q, nw) {
        if (f[q] && pos[q] < nlong) {
            wlong[pos[q]] = wl[q];
            cmode[wl[q]] = 1;
        }
    }
}

__global__ void k_coin_blocked(const int32_t *cand, const int32_t *comm, int64_t K,
                               const int32_t *status, const int32_t *first_commit,
                               int32_t *out) {
    GS_LOOP(k, K) {
        if (status[k] != ST_COIN) continue;
        // reached (frm clean at k) and lost the coin: detector.py:489-493
        if (first_commit[comm[cand[k]]] > (int32_t)k) atomicOr(&out[0], 1);
    }
}

__global__ void k_commit_flags(int64_t K, const int32_t *status, int32_t *f) {
    GS_LOOP(k, K) f[k] = status[k] == ST_COMMIT ? 1 : 0;
}
__global__ void k_gather_gains(int64_t K, const int32_t *f, const int32_t *pos, const double *g,
                               double *out) {
    GS_LOOP(k, K) if (f[k]) out[pos[k]] = g[k];
}

// per-call scratch of run_commit, kept across calls (grow-only)
struct CommitScratch {
    DBuf<int4> tl_rec;   // timeline event records
    DBuf<int32_t> big;   // big-tail candidates + count
    DBuf<int32_t> flag, pos, cand;
    DBuf<int32_t> status;
    DBuf<uint8_t> moving;
    DBuf<CandSpec> spec;
    DBuf<int64_t> mvcnt, mvoff;
    DBuf<int32_t> mv_z;
    DBuf<double> mv_u;
    DBuf<int64_t> mv_e;
    DBuf<uint8_t> mv_i;
    DBuf<int32_t> af, apos;
    DBuf<int32_t> lab, cnt, first_commit, wpos, atk, tl_ptr, tl_ev, wl, remaining;
    DBuf<double> So, Si, gbuf;
    DBuf<uint8_t> dirty;
    DBuf<uint32_t> keys, keys_sorted;
    DBuf<int32_t> vals;
    DBuf<int32_t> wf, wp;
    DBuf<int32_t> cf, cpos;
    DBuf<double> gg;
    DBuf<int32_t> lf, lp, wlong;   // long timelines (CTA walkers)
    DBuf<int2> wwait;
    DBuf<uint8_t> cmode;
    // big candidates as work items (integer-weight graphs)
    DBuf<int64_t> bcnt, boff, ri_off, part_be;
    DBuf<int32_t> ri_cnt;
    DBuf<BigItem> bitems;
    DBuf<double> acc_wt, acc_wf, part_bt;
    DBuf<unsigned long long> bctr;
};

void run_commit(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m, const int32_t *d_cstar,
                uint64_t seed, double accept_prob, int64_t level, int64_t sweep, int *improved,
                int64_t *applied, std::vector<double> *gains, uint32_t *wown) {
    cudaStream_t s = ctx->stream;
    CTX_SCRATCH(CommitScratch, CS);
    const int64_t n = G.n, nc = F.n_comms;
    *improved = 0;
    *applied = 0;
    ctx->last_rounds = 0;
    phase_mark(ctx, -1);
    // candidates: cstar != label, ascending (detector.py:473)
    DBuf<int32_t> &flag = CS.flag, &pos = CS.pos, &cand = CS.cand;
    flag.resize(n + 1);
    pos.resize(n + 1);
    CUDA_TRY(cudaMemsetAsync(flag.p + n, 0, 4, s));
    k_cand_flags<<<grid_for(n, 256), 256, 0, s>>>(d_cstar, F.comm.p, n, flag.p);
    dev_exclusive_sum<int32_t, int32_t>(ctx, flag.p, pos.p, n + 1);
    int32_t K = 0;
    CUDA_TRY(cudaMemcpyAsync(&K, pos.p + n, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    ctx->last_candidates = K;
    if (K == 0) return;
    cand.resize(K);
    k_cand_scatter<<<grid_for(n, 256), 256, 0, s>>>(flag.p, pos.p, n, cand.p);
    DBuf<int32_t> &status = CS.status;
    DBuf<uint8_t> &moving = CS.moving;
    status.resize(K);
    moving.resize(n);
    k_coins<<<grid_for(K, 256), 256, 0, s>>>(cand.p, K, mix_key2(seed, level, sweep), accept_prob,
                                             status.p);
    CommitArgs A;
    {
        static const bool no_runs = getenv("SLM_WALK_RUNS") && atoi(getenv("SLM_WALK_RUNS")) == 0;
        A.runs = no_runs ? 0 : 1;
    }
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
    DBuf<CandSpec> &spec = CS.spec;
    spec.resize(K);
    phase_mark(ctx, PH_CAND);
    const bool sprof = ctx->prof && getenv("SLM_PROFILE_SPEC");
    double st_[8] = {0};
    int st_i = 0;
    double st_t = now_ms();
    auto stick = [&]() {
        if (!sprof) return;
        CUDA_TRY(cudaStreamSynchronize(s));
        const double t = now_ms();
        st_[st_i++] = t - st_t;
        st_t = t;
    };
    unsigned GW = grid_for((int64_t)K * 32, 256, SMS() * 32);
    DBuf<int32_t> &big = CS.big;
    big.resize(K + 1);   // [K] = count
    int32_t *nbig = big.p + K;
    CUDA_TRY(cudaMemsetAsync(nbig, 0, 4, s));
    // moving-neighbour list capacities: each accepted candidate's tail entry volume (one
    // scan fills the lists; they need no exact count pass)
    DBuf<int64_t> &mvcnt = CS.mvcnt, &mvoff = CS.mvoff;
    mvcnt.resize(K + 1);
    mvoff.resize(K + 1);
    CUDA_TRY(cudaMemsetAsync(mvcnt.p, 0, (K + 1) * 8, s));
    // (SLM_BIG_VOL overrides the volume threshold; tests force the big path onto small tails)
    const char *bve = getenv("SLM_BIG_VOL");
    const int64_t big_vol = bve ? std::max<int64_t>(1, atoll(bve)) : BIG_VOL;
    k_spec<<<GW, 256, 0, s>>>(A, K, status.p, spec.p, big.p, nbig, mvcnt.p, big_vol);
    // big candidates: work items over the whole GPU on integer-weight graphs (exact atomics),
    // one CTA each otherwise
    static const bool big_cta = getenv("SLM_BIG_CTA") != nullptr;
    const bool big_items = G.integral && !big_cta;
    int64_t NIT = 0;
    int32_t hnbig = 0;
    if (big_items) {
        CUDA_TRY(cudaMemcpyAsync(&hnbig, nbig, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
    if (big_items && hnbig > 0) {
        const unsigned GB_ = (unsigned)std::min<int64_t>(hnbig, SMS() * 8);
        CS.bcnt.resize(hnbig + 1);
        CS.boff.resize(hnbig + 1);
        CUDA_TRY(cudaMemsetAsync(CS.bcnt.p + hnbig, 0, 8, s));
        k_big_count<<<GB_, 256, 0, s>>>(A, big.p, nbig, CS.bcnt.p);
        dev_exclusive_sum<int64_t, int64_t>(ctx, CS.bcnt.p, CS.boff.p, hnbig + 1);
        CUDA_TRY(cudaMemcpyAsync(&NIT, CS.boff.p + hnbig, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        CS.bitems.resize(std::max<int64_t>(1, NIT));
        CS.ri_off.resize(hnbig);
        CS.ri_cnt.resize(hnbig);
        CS.acc_wt.resize(hnbig);
        CS.acc_wf.resize(hnbig);
        CS.part_bt.resize(std::max<int64_t>(1, NIT));
        CS.part_be.resize(std::max<int64_t>(1, NIT));
        CUDA_TRY(cudaMemsetAsync(CS.acc_wt.p, 0, hnbig * 8, s));
        CUDA_TRY(cudaMemsetAsync(CS.acc_wf.p, 0, hnbig * 8, s));
        k_big_fill<<<GB_, 256, 0, s>>>(A, big.p, nbig, CS.boff.p, CS.bitems.p, CS.ri_off.p,
                                       CS.ri_cnt.p);
        k_big_items_spec<<<grid_for(NIT * 32, 256, SMS() * 64), 256, 0, s>>>(
            A, big.p, CS.bitems.p, NIT, CS.acc_wt.p, CS.acc_wf.p, CS.part_bt.p, CS.part_be.p);
        k_big_finish<<<GB_, 256, 0, s>>>(A, big.p, nbig, CS.acc_wt.p, CS.acc_wf.p, CS.part_bt.p,
                                         CS.part_be.p, CS.ri_off.p, CS.ri_cnt.p, spec.p, mvcnt.p);
    } else if (!big_items) {
        k_spec_big<<<SMS() * 4, SPEC_BLOCK, 0, s>>>(A, big.p, nbig, spec.p, mvcnt.p);
    }
    stick();
    CUDA_TRY(cudaMemsetAsync(moving.p, 0, n, s));
    k_mark_moving<<<GW, 256, 0, s>>>(cand.p, F.comm.p, F.on_cycle.p, F.cptr.p, F.pos.p, F.sz.p,
                                     F.order.p, K, status.p, moving.p);
    DBuf<int32_t> &mv_z = CS.mv_z;
    DBuf<double> &mv_u = CS.mv_u;
    DBuf<int64_t> &mv_e = CS.mv_e;
    DBuf<uint8_t> &mv_i = CS.mv_i;

    stick();
    dev_exclusive_sum<int64_t, int64_t>(ctx, mvcnt.p, mvoff.p, K + 1);
    int64_t NMV = 0;
    CUDA_TRY(cudaMemcpyAsync(&NMV, mvoff.p + K, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    mv_z.resize(NMV);
    mv_u.resize(NMV);
    mv_e.resize(NMV);
    mv_i.resize(NMV);
    k_mv_offsets<<<grid_for(K, 256), 256, 0, s>>>(K, status.p, mvoff.p, spec.p);
    k_mv_scan<<<GW, 256, 0, s>>>(A, K, status.p, spec.p, moving.p, 1, nullptr, mv_z.p, mv_u.p,
                                 mv_e.p, mv_i.p);
    if (big_items) {
        if (hnbig > 0) {
            CS.bctr.resize(hnbig);
            CUDA_TRY(cudaMemsetAsync(CS.bctr.p, 0, hnbig * 8, s));
            k_big_items_mv<<<grid_for(NIT * 32, 256, SMS() * 64), 256, 0, s>>>(
                A, big.p, CS.bitems.p, NIT, spec.p, moving.p, CS.bctr.p, mv_z.p, mv_u.p, mv_e.p,
                mv_i.p);
            k_big_mv_finish<<<grid_for(hnbig, 256), 256, 0, s>>>(big.p, nbig, CS.bctr.p, spec.p);
        }
    } else {
        k_mv_scan_big<<<SMS() * 4, SPEC_BLOCK, 0, s>>>(A, big.p, nbig, spec.p, moving.p, 1, nullptr,
                                                     mv_z.p, mv_u.p, mv_e.p, mv_i.p);
    }
    stick();
    // accepted candidates -> (community, k) pairs -> timelines
    DBuf<int32_t> &af = CS.af, &apos = CS.apos;
    af.resize(K + 1);
    apos.resize(K + 1);
    CUDA_TRY(cudaMemsetAsync(af.p + K, 0, 4, s));
    k_acc_flags<<<grid_for(K, 256), 256, 0, s>>>(K, status.p, af.p);
    dev_exclusive_sum<int32_t, int32_t>(ctx, af.p, apos.p, K + 1);
    int32_t NA = 0;
    CUDA_TRY(cudaMemcpyAsync(&NA, apos.p + K, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    ctx->last_accepted = NA;
    // live state
    DBuf<int32_t> &lab = CS.lab, &cnt = CS.cnt, &first_commit = CS.first_commit, &wpos = CS.wpos, &atk = CS.atk, &tl_ptr = CS.tl_ptr, &tl_ev = CS.tl_ev, &wl = CS.wl, &remaining = CS.remaining;
    DBuf<double> &So = CS.So, &Si = CS.Si, &gbuf = CS.gbuf;
    DBuf<uint8_t> &dirty = CS.dirty;
    lab.resize(n);
    cnt.resize(nc);
    first_commit.resize(nc);
    So.resize(nc);
    Si.resize(nc);
    dirty.resize(nc);
    gbuf.resize(K);
    remaining.resize(1);
    CUDA_TRY(cudaMemcpyAsync(lab.p, F.comm.p, n * 4, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(cnt.p, F.count.p, nc * 4, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(So.p, F.S_out.p, nc * 8, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(Si.p, F.S_in.p, nc * 8, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemsetAsync(dirty.p, 0, nc, s));
    CUDA_TRY(cudaMemsetAsync(first_commit.p, 0x7f, nc * 4, s));   // 0x7f7f7f7f > any k
    if (NA > 0) {
        DBuf<uint32_t> &keys = CS.keys, &keys_sorted = CS.keys_sorted;
        DBuf<int32_t> &vals = CS.vals;
        keys.resize(2 * (int64_t)NA);
        keys_sorted.resize(2 * (int64_t)NA);
        vals.resize(2 * (int64_t)NA);
        tl_ev.resize(2 * (int64_t)NA);
        k_acc_pairs<<<grid_for(K, 256), 256, 0, s>>>(cand.p, F.comm.p, d_cstar, K, af.p, apos.p,
                                                     keys.p, vals.p);
        stick();
        CS.tl_rec.resize(2 * (int64_t)NA);
        sort_pairs_u32_i32(ctx, keys.p, keys_sorted.p, vals.p, tl_ev.p, 2 * (int64_t)NA,
                           bits_for(nc + 1));
        tl_ptr.resize(nc + 1);
        k_lb32c<<<grid_for(nc + 1, 256), 256, 0, s>>>(keys_sorted.p, 2 * (int64_t)NA, nc, tl_ptr.p);
        k_ev_rec<<<grid_for(2 * (int64_t)NA, 256), 256, 0, s>>>(tl_ev.p, 2 * (int64_t)NA, cand.p,
                                                               F.comm.p, d_cstar, CS.tl_rec.p);
        // walkers: communities with a non-empty timeline
        DBuf<int32_t> &wf = CS.wf, &wp = CS.wp;
        wf.resize(nc + 1);
        wp.resize(nc + 1);
        wpos.resize(nc);
        atk.resize(nc);
        CS.wwait.resize(nc);
        CUDA_TRY(cudaMemsetAsync(CS.wwait.p, 0xff, nc * sizeof(int2), s));   // {-1, -1}
        CUDA_TRY(cudaMemsetAsync(wf.p + nc, 0, 4, s));
        k_walker_list<<<grid_for(nc, 256), 256, 0, s>>>(tl_ptr.p, nc, wf.p);
        dev_exclusive_sum<int32_t, int32_t>(ctx, wf.p, wp.p, nc + 1);
        int32_t NW = 0;
        CUDA_TRY(cudaMemcpyAsync(&NW, wp.p + nc, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        wl.resize(NW);
        stick();
        k_walker_scatter<<<grid_for(nc, 256), 256, 0, s>>>(wf.p, wp.p, tl_ptr.p, CS.tl_rec.p, nc,
                                                           wl.p, wpos.p, atk.p, CS.wwait.p);
        CUDA_TRY(cudaMemcpyAsync(remaining.p, &NA, 4, cudaMemcpyHostToDevice, s));
        Live V;
        V.lab = lab.p;
        V.S_out = So.p;
        V.S_in = Si.p;
        V.cnt = cnt.p;
        V.dirty = dirty.p;
        V.first_commit = first_commit.p;
        V.a = F.a.p;   // committed pointers are written in place (tails come from the layout)
        V.wpos = wpos.p;
        V.atk = atk.p;
        V.wwait = CS.wwait.p;
        V.tl_ptr = tl_ptr.p;
        V.tl_ev = tl_ev.p;
        V.tl_rec = CS.tl_rec.p;
        V.mv.z = mv_z.p;
        V.mv.u = mv_u.p;
        V.mv.e = mv_e.p;
        V.mv.is_i = mv_i.p;
        V.gain = gbuf.p;
        V.remaining = remaining.p;
        stick();
        if (sprof)
            fprintf(stderr, "[spec] K=%d NA=%d: spec %.2f mark+mvcount %.2f fill+acc %.2f state+pairs %.2f "
                    "sort+walkers %.2f scatter %.2f ms\n", K, NA, st_[0], st_[1], st_[2], st_[3],
                    st_[4], st_[5]);
        phase_mark(ctx, PH_SPEC);
        const unsigned GWK = grid_for((int64_t)NW * 32, 256, SMS() * 64);
        int32_t rem = NA;
        std::vector<double> rt;
        const bool wprof = ctx->prof && getenv("SLM_PROFILE_WALK");
        CTX_SCRATCH(DBuf<unsigned long long>, wst);
        V.wst = nullptr;
        std::vector<std::string> rinfo;
        if (wprof) {
            wst.resize(8);
            V.wst = wst.p;
        }
        // one persistent launch on a resident grid (SLM_WALK_ROUNDS=1: relaunch per round)
        // walkers park and spin on verdicts of other blocks, so the persistent grid must be
        // co-resident: occupancy x the device's SMs, launched cooperatively (the launch fails
        // instead of deadlocking when the grid cannot be resident, e.g. under MPS limits;
        // then this call falls back to one launch per round)
        if (ctx->walk_blocks == 0) {
            int per_sm = 0;
            CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_walk, WALK_BLOCK, 0));
            ctx->walk_blocks = std::max(1, per_sm) * ctx->num_sms;
        }
        bool rounds_mode = getenv("SLM_WALK_ROUNDS") != nullptr;
        const unsigned GWP = (unsigned)std::min<int64_t>(GWK, ctx->walk_blocks);
        // timelines longer than LONG_TL events (hub communities) are walked by whole CTAs,
        // blocks [0, nlong) of the persistent grid (at most 16: the rest walk the many short
        // timelines of the early sweeps)
        static const int LONG_TL = getenv("SLM_WALK_LONG") ? std::max(32, atoi(getenv("SLM_WALK_LONG")))
                                                           : 8192;
        int32_t nlong = 0;
        const uint8_t *cmode = nullptr;
        if (!rounds_mode && NW > 0) {
            DBuf<int32_t> &lf = CS.lf, &lp = CS.lp;
            lf.resize(NW + 1);
            lp.resize(NW + 1);
            CUDA_TRY(cudaMemsetAsync(lf.p + NW, 0, 4, s));
            k_long_flags<<<grid_for(NW, 256), 256, 0, s>>>(wl.p, NW, tl_ptr.p, LONG_TL, lf.p);
            dev_exclusive_sum<int32_t, int32_t>(ctx, lf.p, lp.p, NW + 1);
            int32_t NL = 0;
            CUDA_TRY(cudaMemcpyAsync(&NL, lp.p + NW, 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            nlong = std::min<int32_t>(NL, std::min<int32_t>(16, (int32_t)(GWP / 8)));
            if (nlong > 0) {
                CS.cmode.resize(nc);
                CS.wlong.resize(nlong);
                CUDA_TRY(cudaMemsetAsync(CS.cmode.p, 0, nc, s));
                k_long_scatter<<<grid_for(NW, 256), 256, 0, s>>>(lf.p, lp.p, wl.p, NW, nlong,
                                                                 CS.wlong.p, CS.cmode.p);
                cmode = CS.cmode.p;
            }
        }
        for (int round = 0; rem > 0; round++) {
            if (wprof) CUDA_TRY(cudaMemsetAsync(wst.p, 0, 64, s));
            const double t0 = ctx->prof ? now_ms() : 0.0;
            if (rounds_mode)
                k_walk<<<GWK, WALK_BLOCK, 0, s>>>(A, V, wl.p, NW, status.p, spec.p, 0, nullptr, 0,
                                                  nullptr);
            else {
                int one = 1;
                int64_t nw64 = NW;
                const int32_t *wlp = wl.p, *wlg = CS.wlong.p;
                int32_t *stp = status.p;
                const CandSpec *spp = spec.p;
                void *kargs[] = {(void *)&A, (void *)&V, (void *)&wlp, (void *)&nw64, (void *)&stp,
                                 (void *)&spp, (void *)&one, (void *)&wlg, (void *)&nlong,
                                 (void *)&cmode};
                cudaError_t le = cudaLaunchCooperativeKernel((const void *)k_walk, dim3(GWP),
                                                             dim3(WALK_BLOCK), kargs, 0, s);
                if (le != cudaSuccess) {
                    cudaGetLastError();
                    rounds_mode = true;
                    k_walk<<<GWK, WALK_BLOCK, 0, s>>>(A, V, wl.p, NW, status.p, spec.p, 0, nullptr,
                                                      0, nullptr);
                }
            }
            CUDA_TRY(cudaMemcpyAsync(&rem, remaining.p, 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            if (ctx->prof) rt.push_back(now_ms() - t0);
            if (wprof) {
                unsigned long long h[8];
                CUDA_TRY(cudaMemcpy(h, wst.p, 64, cudaMemcpyDeviceToHost));
                char buf[160];
                snprintf(buf, sizeof buf, "[%.2fms ev %llu max %llu w %llu rp %llu/%llu tl %llu "
                         "maxcommit %llu maxbarrier %llu]",
                         rt.back(), h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
                rinfo.push_back(buf);
            }
            ctx->last_rounds = round + 1;
            SLM_REQUIRE(round < 10000000, SLM_ESTATE, "commit walkers made no progress");
        }
        if (ctx->prof && getenv("SLM_PROFILE_WALK")) {
            fprintf(stderr, "walk K=%d NA=%d NW=%d rounds=%zu ms:", K, NA, NW, rt.size());
            for (size_t q = 0; q < rinfo.size(); q++) fprintf(stderr, " %s", rinfo[q].c_str());
            double tot = 0;
            for (double x : rt) tot += x;
            fprintf(stderr, " total %.2f\n", tot);
        }
    }
    phase_mark(ctx, PH_WALK);
    int32_t *dflags = ctx->i32d.resize(4);
    CUDA_TRY(cudaMemsetAsync(dflags, 0, 4, s));
    const unsigned GK = grid_for(K, 256);
    k_coin_blocked<<<GK, 256, 0, s>>>(cand.p, F.comm.p, K, status.p, first_commit.p, dflags);
    // applied + gains in ascending candidate order
    DBuf<int32_t> &cf = CS.cf, &cpos = CS.cpos;
    cf.resize(K + 1);
    cpos.resize(K + 1);
    CUDA_TRY(cudaMemsetAsync(cf.p + K, 0, 4, s));
    k_commit_flags<<<GK, 256, 0, s>>>(K, status.p, cf.p);
    dev_exclusive_sum<int32_t, int32_t>(ctx, cf.p, cpos.p, K + 1);
    int32_t hv[2] = {0, 0};
    CUDA_TRY(cudaMemcpyAsync(&hv[0], cpos.p + K, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&hv[1], dflags, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *applied = hv[0];
    *improved = (hv[0] > 0) || hv[1];
    // own-community sums follow the moved nodes (F.comm: labels before the commit, lab: after)
    if (wown && hv[0] > 0) {
        wown_to_node_order(ctx, G);
        commit_wown_deltas(ctx, G, F.comm.p, CS.lab.p, wown);
    }
    if (gains && hv[0] > 0) {
        DBuf<double> &gg = CS.gg;
        gg.resize(hv[0]);
        k_gather_gains<<<GK, 256, 0, s>>>(K, cf.p, cpos.p, gbuf.p, gg.p);
        gains->resize(hv[0]);
        CUDA_TRY(cudaMemcpyAsync(gains->data(), gg.p, hv[0] * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
}

// ---- own-community group sums across a commit: w_own[z] changes only for the neighbours of
// moved nodes (a move a -> b of v takes u(z, v) from z's sum when z sits in a, adds it when z
// sits in b); a moved node's sum is recomputed over its row.  uint32 wrap-around arithmetic is
// exact whatever the order of the atomic updates.
__global__ void k_wown_flags(const int32_t *pre, const int32_t *post, int64_t n, int32_t *f) {
    GS_LOOP(i, n) f[i] = pre[i] != post[i] ? 1 : 0;
}
__global__ void k_wown_list(const int32_t *f, const int32_t *pos, int64_t n, int32_t *list) {
    GS_LOOP(i, n) if (f[i]) list[pos[i]] = (int32_t)i;
}
__global__ void k_wown_delta(const int64_t *uptr, const int32_t *unbr, const uint32_t *u32,
                             const int32_t *pre, const int32_t *post, const int32_t *moved,
                             const int32_t *list, int64_t nm, uint32_t *wown) {
    const int lane = threadIdx.x & 31;
    for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < nm;
         q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t v = list[q];
        const int32_t a = pre[v], b = post[v];
        uint32_t own = 0;
        for (int64_t e = uptr[v] + lane; e < uptr[v + 1]; e += 32) {
            const int32_t z = unbr[e];
            const uint32_t u = u32[e];
            const int32_t pz = post[z];
            if (pz == b) own += u;
            if (moved[z]) continue;   // recomputed by its own warp
            if (pz == a) atomicSub(wown + z, u);
            else if (pz == b) atomicAdd(wown + z, u);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) own += __shfl_xor_sync(0xffffffffu, own, off);
        if (lane == 0) wown[v] = own;
    }
}
void commit_wown_deltas(slm_ctx *ctx, const LevelGraph &G, const int32_t *pre, const int32_t *post,
                        uint32_t *wown) {
    cudaStream_t s = ctx->stream;
    const int64_t n = G.n;
    CTX_SCRATCH(DBuf<int32_t>, f);   // grow-only scratch kept across calls
    CTX_SCRATCH(DBuf<int32_t>, pos);
    CTX_SCRATCH(DBuf<int32_t>, list);
    f.resize(n + 1);
    pos.resize(n + 1);
    CUDA_TRY(cudaMemsetAsync(f.p + n, 0, 4, s));
    k_wown_flags<<<grid_for(n, 256), 256, 0, s>>>(pre, post, n, f.p);
    dev_exclusive_sum<int32_t, int32_t>(ctx, f.p, pos.p, n + 1);
    int32_t nm = 0;
    CUDA_TRY(cudaMemcpyAsync(&nm, pos.p + n, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (nm == 0) return;
    list.resize(nm);
    k_wown_list<<<grid_for(n, 256), 256, 0, s>>>(f.p, pos.p, n, list.p);
    k_wown_delta<<<grid_for((int64_t)nm * 32, 256), 256, 0, s>>>(G.uptr.p, G.unbr.p, G.uu32.p, pre,
                                                                post, f.p, list.p, nm, wown);
    CUDA_TRY(cudaGetLastError());
}

// a kernel of this translation unit (module preloading, slm_capi.cu preload_modules)
const void *slm_anchor_commit() { return (const void *)k_cand_flags; }
