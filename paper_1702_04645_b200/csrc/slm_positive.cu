// slm_positive.cu -- POSITIVE correction (positive_correction, detector.py:338-362;
// _split_community 197-285; _detach_gain 178-194; _best_pair_cut 288-335).
//
// A bad community (a member with negative local gain) is split repeatedly by its best
// strictly positive single cut.  Parts are independent (each split touches only its part),
// so the reference's LIFO stack order matters only for the order of the gains list, which
// is reconstructed exactly on the host.  Two executors:
//
//  * small parts (<= SMALL_PART members): one warp per part, replaying the reference's LIFO
//    stack.  Parts are contiguous slices of the community's DFS pre-order (slm_forest.cu);
//    every branch-cut gain of a part comes from one pass:
//        x_w(sub(x)) = sum_{v in sub(x)} dep[v],
//        dep[v] = w_part(v) - sum_{entries (y,z) with LCA(y,z) = v} u,
//    with prefix sums over the slice for the subtree sums and the reference's fp64 operand
//    order for the gain.  The cut is the first strict maximum > 0 in ascending node id; a
//    2-cycle pair cut (cycles are <= 2) equals detaching the DFS subtree of the
//    cycle's second node with both cycle nodes self-assigned.
//
//  * giant parts (R-MAT hub communities reach ~10^6 members and thousands of sequential
//    splits): grid-wide kernels with incremental state.  After the first full pass, a cut
//    of subtree b only changes the part totals, the subtree sums of b's ancestors, and the
//    crossing weights x_w along the tree paths of the edges between b and the rest, so a
//    split costs O(|part|) gain evaluations plus O(edges(b) * depth) updates instead of a
//    full O(edges(part)) recomputation.  Subtree ranges keep the community's original DFS
//    coordinates; removed members are masked by their part id.
#include "slm_internal.cuh"
#include <cub/cub.cuh>
#include <algorithm>
#include <cstring>
#include <cstdlib>

// parts up to this size use the warp executor; SLM_SMALL_PART overrides it (tests force the
// giant executor onto small graphs with it)
static int SMALL_PART = 4096;
static void read_small_part() {
    const char *e = getenv("SLM_SMALL_PART");
    SMALL_PART = e ? std::max(1, atoi(e)) : 4096;
}

#define GS_LOOP(i, n)                                                                      \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n);              \
         i += (int64_t)gridDim.x * blockDim.x)

struct PartDesc {
    int32_t off;          // region start in pbuf / sstk / gains
    int32_t len;          // members
    int32_t from_layout;  // 1: copy order[off..) and sz; 0: pbuf/psz pre-filled
    int32_t pad;
};

struct PosArgs {
    const int64_t *uptr;
    const int32_t *unbr;
    const double *uu;
    const double *s_out, *s_in;
    int32_t *a;
    const int32_t *order, *sz0;
    const PartDesc *parts;
    int64_t nparts;
    double m, m2;
    int32_t *pbuf, *tbuf, *pmark, *ppos, *psz;
    int2 *sstk;
    double *wpart, *dep, *pre_so, *pre_si, *pre_dep;
    double *gains;       // per part region
    int32_t *ngains;     // per part
    int32_t *neg_unres;  // per part
    uint32_t *stamp_ctr;
    int32_t *flags;      // [0] changed, [1] unsupported cycle
};

__device__ __forceinline__ double wsum_d(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}
__device__ __forceinline__ int wsum_i(int v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// exclusive prefix over a slice, written at out[k]; returns the total
__device__ double warp_exscan(const int32_t *P, int len, const double *val_of_node, double *out) {
    const int lane = threadIdx.x & 31;
    double carry = 0.0;
    for (int cb = 0; cb < len; cb += 32) {
        int k = cb + lane;
        double v = 0.0;
        if (k < len) v = val_of_node[P[k]];
        double inc = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            double o = __shfl_up_sync(0xffffffffu, inc, off);
            if (lane >= off) inc += o;
        }
        if (k < len) out[k] = carry + (inc - v);
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    return carry;
}

// w_part of each member: lanes take members; long rows are handled warp-wide afterwards
__device__ void member_weights(const PosArgs &A, const int32_t *P, int len, uint32_t stamp) {
    const int lane = threadIdx.x & 31;
    for (int cb = 0; cb < len; cb += 32) {
        int k = cb + lane;
        bool longrow = false;
        if (k < len) {
            int32_t x = P[k];
            int64_t e0 = A.uptr[x], e1 = A.uptr[x + 1];
            if (e1 - e0 > 64) {
                longrow = true;
            } else {
                double wp = 0.0;
                for (int64_t e = e0; e < e1; e++)
                    if (A.pmark[A.unbr[e]] == (int32_t)stamp) wp += A.uu[e];
                A.wpart[x] = wp;
                A.dep[x] = wp;
            }
        }
        unsigned lm = __ballot_sync(0xffffffffu, longrow);
        while (lm) {
            int src = __ffs(lm) - 1;
            lm &= lm - 1;
            int32_t x = P[cb + src];
            double wp = 0.0;
            for (int64_t e = A.uptr[x] + lane; e < A.uptr[x + 1]; e += 32)
                if (A.pmark[A.unbr[e]] == (int32_t)stamp) wp += A.uu[e];
            wp = wsum_d(wp);
            if (lane == 0) {
                A.wpart[x] = wp;
                A.dep[x] = wp;
            }
        }
    }
}

__global__ void __launch_bounds__(128) k_positive(PosArgs A) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double m = A.m, m2 = A.m2;
    for (int64_t bi = w; bi < A.nparts; bi += nw) {
        const PartDesc D = A.parts[bi];
        const int32_t base = D.off, size = D.len;
        if (D.from_layout) {
            for (int k = lane; k < size; k += 32) {
                int32_t x = A.order[base + k];
                A.pbuf[base + k] = x;
                A.psz[x] = A.sz0[x];
            }
        }
        int sp = 0;
        if (lane == 0) A.sstk[base] = make_int2(0, size);
        sp = 1;
        int ng = 0, unres = 0;
        __syncwarp();
        while (sp > 0) {
            sp--;
            const int2 seg = A.sstk[base + sp];
            const int off = seg.x, len = seg.y;
            if (len <= 1) continue;
            int32_t *P = A.pbuf + base + off;
            uint32_t stamp = 0;
            if (lane == 0) stamp = atomicAdd(A.stamp_ctr, 1u) + 1u;
            stamp = __shfl_sync(0xffffffffu, stamp, 0);
            for (int k = lane; k < len; k += 32) {
                int32_t x = P[k];
                A.pmark[x] = (int32_t)stamp;
                A.ppos[x] = k;
            }
            __syncwarp();
            double so_c = 0.0, si_c = 0.0;
            for (int k = lane; k < len; k += 32) {
                so_c += A.s_out[P[k]];
                si_c += A.s_in[P[k]];
            }
            so_c = wsum_d(so_c);
            si_c = wsum_d(si_c);
            member_weights(A, P, len, stamp);
            __syncwarp();
            // member gains against the part (detector.py:217-223)
            int neg = 0;
            for (int k = lane; k < len; k += 32) {
                int32_t x = P[k];
                const double sox = A.s_out[x], six = A.s_in[x];
                double g = A.wpart[x] / m - (sox * (si_c - six) + six * (so_c - sox)) / m2;
                if (g < 0.0) neg++;
            }
            neg = wsum_i(neg);
            if (neg == 0) continue;
            const int32_t r = P[0];
            const int32_t q = A.a[r];
            const bool two = (q != r);
            if (two && A.a[q] != r) {   // cycle longer than 2: not produced by SLM (F5)
                if (lane == 0) atomicOr(&A.flags[1], 1);
                continue;
            }
            __syncwarp();
            // LCA deposits: -u at the lowest ancestor of y whose DFS range holds z
            for (int k = lane; k < len; k += 32) {
                int32_t y = P[k];
                for (int64_t e = A.uptr[y]; e < A.uptr[y + 1]; e++) {
                    int32_t z = A.unbr[e];
                    if (A.pmark[z] != (int32_t)stamp) continue;
                    int32_t pz = A.ppos[z];
                    int32_t anc = y;
                    for (;;) {
                        int32_t pa = A.ppos[anc];
                        if (pz >= pa && pz < pa + A.psz[anc]) break;
                        anc = A.a[anc];
                    }
                    atomicAdd(&A.dep[anc], -A.uu[e]);
                }
            }
            __syncwarp();
            double *pso = A.pre_so + base + off, *psi = A.pre_si + base + off,
                   *pdp = A.pre_dep + base + off;
            double tso = warp_exscan(P, len, A.s_out, pso);
            double tsi = warp_exscan(P, len, A.s_in, psi);
            double tdp = warp_exscan(P, len, A.dep, pdp);
            __syncwarp();
            // branch cuts over non-cycle members (detector.py:238-253)
            double bg = -INFINITY;
            int32_t bx = 0x7fffffff;
            for (int k = lane; k < len; k += 32) {
                int32_t x = P[k];
                if (x == r || (two && x == q)) continue;
                int hi = k + A.psz[x];
                double so_b = (hi == len ? tso : pso[hi]) - pso[k];
                double si_b = (hi == len ? tsi : psi[hi]) - psi[k];
                double x_w = (hi == len ? tdp : pdp[hi]) - pdp[k];
                double null = -so_c * si_b - so_b * si_c + 2.0 * so_b * si_b;
                double gain = -x_w / m - null / (m * m);
                if (gain > bg || (gain == bg && x < bx)) {
                    bg = gain;
                    bx = x;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                double og = __shfl_xor_sync(0xffffffffu, bg, o);
                int32_t ox = __shfl_xor_sync(0xffffffffu, bx, o);
                if (og > bg || (og == bg && ox < bx)) {
                    bg = og;
                    bx = ox;
                }
            }
            int32_t cut_x = -1;
            bool pair = false;
            double gain = 0.0;
            if (bx != 0x7fffffff && bg > 0.0) {
                cut_x = bx;
                gain = bg;
            } else if (two) {
                // pair cut (detector.py:254-274, 288-335 with s = 2)
                int k = A.ppos[q];
                int hi = k + A.psz[q];
                double so_b = (hi == len ? tso : pso[hi]) - pso[k];
                double si_b = (hi == len ? tsi : psi[hi]) - psi[k];
                double x_w = (hi == len ? tdp : pdp[hi]) - pdp[k];
                double null = -so_c * si_b - so_b * si_c + 2.0 * so_b * si_b;
                double pg = -x_w / m - null / m2;
                if (pg > 0.0) {
                    cut_x = q;
                    pair = true;
                    gain = pg;
                }
            }
            if (cut_x < 0) {
                unres += neg;   // detector.py:275-277
                continue;
            }
            const int lo = A.ppos[cut_x];
            const int sx = A.psz[cut_x];
            if (lane == 0) {
                A.gains[base + ng] = gain;
                if (pair) {
                    A.a[r] = r;
                    A.a[q] = q;
                    A.psz[r] -= sx;
                } else {
                    int32_t anc = A.a[cut_x];
                    A.a[cut_x] = cut_x;
                    for (;;) {
                        A.psz[anc] -= sx;
                        if (anc == r) break;
                        anc = A.a[anc];
                    }
                }
                A.flags[0] = 1;
            }
            ng++;
            // rearrange slice: rest (DFS order) then the cut subtree
            for (int k = lane; k < len; k += 32) {
                int src;
                if (k < lo) src = k;
                else if (k < len - sx) src = k + sx;
                else src = k - (len - sx) + lo;
                A.tbuf[base + off + k] = P[src];
            }
            __syncwarp();
            for (int k = lane; k < len; k += 32) P[k] = A.tbuf[base + off + k];
            if (lane == 0) {
                A.sstk[base + sp] = make_int2(off, len - sx);
                A.sstk[base + sp + 1] = make_int2(off + len - sx, sx);
            }
            sp += 2;
            __syncwarp();
        }
        if (lane == 0) {
            A.ngains[bi] = ng;
            A.neg_unres[bi] = unres;
        }
    }
}

// =========================================================== giant-part executor

struct GiantArgs {
    const int64_t *uptr;
    const int32_t *unbr;
    const double *uu;
    const double *s_out, *s_in;
    int32_t *a;
    const int32_t *order, *pos, *sz;   // community layout (original coordinates)
    int32_t *gmark;
    double *wpart, *dep, *xw, *sob, *sib;
    double m, m2;
};

struct GiantState {          // device-resident scalars of the current giant part
    double so_c, si_c;
    int32_t pid, root, q, two;
    // eval result
    int32_t neg;
    int32_t best_x;
    double best_gain;
    double pair_gain;
    int32_t bsize;
    int32_t pad;
};

// members of a giant part: order[lo..hi) with gmark == pid
__global__ void k_g_mark(const int32_t *order, int64_t lo, int64_t hi, int32_t pid, int32_t *gmark) {
    for (int64_t k = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < hi;
         k += (int64_t)gridDim.x * blockDim.x)
        gmark[order[k]] = pid;
}

// warp per member: w_part and dep (= w_part before LCA deposits)
__global__ void k_g_wpart(GiantArgs A, int64_t lo, int64_t hi, int32_t pid) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = lo + w; k < hi; k += nw) {
        int32_t x = A.order[k];
        if (A.gmark[x] != pid) continue;
        double wp = 0.0;
        for (int64_t e = A.uptr[x] + lane; e < A.uptr[x + 1]; e += 32)
            if (A.gmark[A.unbr[e]] == pid) wp += A.uu[e];
        wp = wsum_d(wp);
        if (lane == 0) {
            A.wpart[x] = wp;
            A.dep[x] = wp;
        }
    }
}

__device__ __forceinline__ bool in_range(const GiantArgs &A, int32_t anc, int32_t pz) {
    int32_t pa = A.pos[anc];
    return pz >= pa && pz < pa + A.sz[anc];
}

__global__ void k_g_lca(GiantArgs A, int64_t lo, int64_t hi, int32_t pid) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = lo + w; k < hi; k += nw) {
        int32_t y = A.order[k];
        if (A.gmark[y] != pid) continue;
        for (int64_t e = A.uptr[y] + lane; e < A.uptr[y + 1]; e += 32) {
            int32_t z = A.unbr[e];
            if (A.gmark[z] != pid) continue;
            int32_t pz = A.pos[z];
            int32_t anc = y;
            while (!in_range(A, anc, pz)) anc = A.a[anc];
            atomicAdd(&A.dep[anc], -A.uu[e]);
        }
    }
}

__global__ void k_g_gather(GiantArgs A, int64_t lo, int64_t hi, int32_t pid, double *vso,
                           double *vsi, double *vdp) {
    for (int64_t k = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < hi;
         k += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = A.order[k];
        bool in = A.gmark[x] == pid;
        vso[k - lo] = in ? A.s_out[x] : 0.0;
        vsi[k - lo] = in ? A.s_in[x] : 0.0;
        vdp[k - lo] = in ? A.dep[x] : 0.0;
    }
}

// subtree sums in original coordinates: index of node x in the part slice = cbase+pos-lo
__global__ void k_g_subsums(GiantArgs A, int64_t lo, int64_t hi, int64_t cbase, int32_t pid,
                            const double *pso, const double *psi, const double *pdp,
                            GiantState *S) {
    for (int64_t k = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < hi;
         k += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = A.order[k];
        if (A.gmark[x] != pid) continue;
        int64_t i0 = cbase + A.pos[x] - lo, i1 = i0 + A.sz[x];
        A.sob[x] = pso[i1] - pso[i0];
        A.sib[x] = psi[i1] - psi[i0];
        A.xw[x] = pdp[i1] - pdp[i0];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        S->so_c = pso[hi - lo];
        S->si_c = psi[hi - lo];
    }
}

constexpr int GE_BLOCK = 256;

__global__ void __launch_bounds__(GE_BLOCK) k_g_eval(GiantArgs A, int64_t lo, int64_t hi,
                                                     const GiantState *S, int32_t *blk_neg,
                                                     double *blk_g, int32_t *blk_x) {
    __shared__ double sg[GE_BLOCK / 32];
    __shared__ int32_t sx[GE_BLOCK / 32];
    __shared__ int32_t sn[GE_BLOCK / 32];
    const double m = A.m, m2 = A.m2;
    const double so_c = S->so_c, si_c = S->si_c;
    const int32_t pid = S->pid, r = S->root, q = S->q;
    const bool two = S->two;
    double bg = -INFINITY;
    int32_t bx = 0x7fffffff;
    int neg = 0;
    for (int64_t k = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < hi;
         k += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = A.order[k];
        if (A.gmark[x] != pid) continue;
        const double sox = A.s_out[x], six = A.s_in[x];
        double g = A.wpart[x] / m - (sox * (si_c - six) + six * (so_c - sox)) / m2;
        if (g < 0.0) neg++;
        if (x == r || (two && x == q)) continue;
        double so_b = A.sob[x], si_b = A.sib[x];
        double null = -so_c * si_b - so_b * si_c + 2.0 * so_b * si_b;
        double gain = -A.xw[x] / m - null / (m * m);
        if (gain > bg || (gain == bg && x < bx)) {
            bg = gain;
            bx = x;
        }
    }
    neg = wsum_i(neg);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double og = __shfl_xor_sync(0xffffffffu, bg, o);
        int32_t ox = __shfl_xor_sync(0xffffffffu, bx, o);
        if (og > bg || (og == bg && ox < bx)) {
            bg = og;
            bx = ox;
        }
    }
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sg[wid] = bg;
        sx[wid] = bx;
        sn[wid] = neg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double g0 = sg[0];
        int32_t x0 = sx[0];
        int nn = sn[0];
        for (int i = 1; i < GE_BLOCK / 32; i++) {
            nn += sn[i];
            if (sg[i] > g0 || (sg[i] == g0 && sx[i] < x0)) {
                g0 = sg[i];
                x0 = sx[i];
            }
        }
        blk_g[blockIdx.x] = g0;
        blk_x[blockIdx.x] = x0;
        blk_neg[blockIdx.x] = nn;
    }
}

__global__ void k_g_reduce(GiantArgs A, int nb, const int32_t *blk_neg, const double *blk_g,
                           const int32_t *blk_x, GiantState *S) {
    if (threadIdx.x != 0) return;
    double g0 = -INFINITY;
    int32_t x0 = 0x7fffffff;
    int nn = 0;
    for (int i = 0; i < nb; i++) {
        nn += blk_neg[i];
        if (blk_g[i] > g0 || (blk_g[i] == g0 && blk_x[i] < x0)) {
            g0 = blk_g[i];
            x0 = blk_x[i];
        }
    }
    S->neg = nn;
    S->best_gain = g0;
    S->best_x = x0;
    S->pair_gain = -INFINITY;
    if (S->two) {
        const double m = A.m, m2 = A.m2;
        const int32_t q = S->q;
        double so_b = A.sob[q], si_b = A.sib[q];
        double so_c = S->so_c, si_c = S->si_c;
        double null = -so_c * si_b - so_b * si_c + 2.0 * so_b * si_b;
        S->pair_gain = -A.xw[q] / m - null / m2;
    }
}

// re-mark the cut subtree as part pid_b and count it
__global__ void k_g_cut_mark(GiantArgs A, int64_t cbase, int32_t xc, int32_t pid, int32_t pid_b,
                             GiantState *S) {
    const int64_t lo = cbase + A.pos[xc], hi = lo + A.sz[xc];
    int cnt = 0;
    for (int64_t k = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < hi;
         k += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = A.order[k];
        if (A.gmark[x] == pid) {
            A.gmark[x] = pid_b;
            cnt++;
        }
    }
    cnt = wsum_i(cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&S->bsize, cnt);
}

// one thread: apply the cut to a, the part totals and the ancestors' subtree sums
__global__ void k_g_apply(GiantArgs A, int32_t xc, int32_t pair, GiantState *S) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int32_t r = S->root;
    const double sb = A.sob[xc], ib = A.sib[xc];
    S->so_c -= sb;
    S->si_c -= ib;
    if (pair) {
        A.sob[r] -= sb;
        A.sib[r] -= ib;
        A.a[r] = r;
        A.a[xc] = xc;
        S->two = 0;
    } else {
        int32_t y = A.a[xc];
        A.a[xc] = xc;
        for (;;) {
            A.sob[y] -= sb;
            A.sib[y] -= ib;
            if (y == r) break;
            y = A.a[y];
        }
    }
}

// edges between the cut subtree b and the rest R: drop them from w_part (R side) and from
// x_w along the tree path between their endpoints (strictly below the LCA, R nodes only)
__global__ void k_g_cross(GiantArgs A, int64_t cbase, int32_t xc, int32_t xc_parent, int32_t pid,
                          int32_t pid_b) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t lo = cbase + A.pos[xc], hi = lo + A.sz[xc];
    for (int64_t k = lo + w; k < hi; k += nw) {
        int32_t z = A.order[k];
        if (A.gmark[z] != pid_b) continue;
        const int32_t pz = A.pos[z];
        for (int64_t e = A.uptr[z] + lane; e < A.uptr[z + 1]; e += 32) {
            int32_t v = A.unbr[e];
            if (A.gmark[v] != pid) continue;
            const double u = A.uu[e];
            atomicAdd(&A.wpart[v], -u);
            int32_t y = v;
            while (!in_range(A, y, pz)) {
                atomicAdd(&A.xw[y], -u);
                y = A.a[y];
            }
            const int32_t lca = y;
            y = xc_parent;
            while (y != lca) {
                atomicAdd(&A.xw[y], -u);
                y = A.a[y];
            }
        }
    }
}

// compact a (small) cut subtree into its own descriptor region with in-part subtree sizes
__global__ void k_g_compact_flags(const int32_t *order, const int32_t *gmark, int64_t lo,
                                  int64_t hi, int32_t pid_b, int32_t *flag) {
    for (int64_t k = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < hi;
         k += (int64_t)gridDim.x * blockDim.x)
        flag[k - lo] = gmark[order[k]] == pid_b ? 1 : 0;
}
__global__ void k_g_compact_fill(const int32_t *order, const int32_t *pos, const int32_t *flag,
                                 const int32_t *idx, int64_t lo, int64_t hi, int32_t dst_off,
                                 int32_t *pbuf, int32_t *posb) {
    for (int64_t k = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < hi;
         k += (int64_t)gridDim.x * blockDim.x)
        if (flag[k - lo]) {
            pbuf[dst_off + idx[k - lo]] = order[k];
            posb[idx[k - lo]] = pos[order[k]];
        }
}
__global__ void k_g_compact_psz(const int32_t *pbuf, const int32_t *posb, const int32_t *sz,
                                int32_t dst_off, int32_t len, int32_t *psz) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t y = pbuf[dst_off + i];
        int32_t endp = posb[i] + sz[y];
        int32_t lo = (int32_t)i, hi = len;   // first index with posb >= endp
        while (lo < hi) {
            int32_t mid = (lo + hi) >> 1;
            if (posb[mid] < endp) lo = mid + 1;
            else hi = mid;
        }
        psz[y] = lo - (int32_t)i;
    }
}

__global__ void k_bad_flags(const uint8_t *bad, int64_t nc, int32_t *f) {
    GS_LOOP(c, nc) f[c] = bad[c] ? 1 : 0;
}
__global__ void k_bad_scatter(const int32_t *f, const int32_t *pos, int64_t nc, int32_t *list) {
    GS_LOOP(c, nc) if (f[c]) list[pos[c]] = (int32_t)c;
}
__global__ void k_init_i32(int32_t *x, int64_t n, int32_t v) { GS_LOOP(i, n) x[i] = v; }

static DBuf<uint32_t> g_stamp;   // monotone part stamps (never reset)

namespace {

struct Split {              // one cut of a giant part
    double gain;
    int kind;               // 0: small child (descriptor index), 1: giant child (giant id)
    int64_t child;
};
struct GiantRec {
    std::vector<Split> splits;
};

struct PosCtx {
    slm_ctx *ctx;
    const LevelGraph *G;
    Forest *F;
    double m;
    GiantArgs GA;
    DBuf<GiantState> S;
    DBuf<int32_t> blk_neg, blk_x, cflag, cidx;
    DBuf<double> blk_g, vso, vsi, vdp, pso, psi, pdp;
    int32_t next_pid = 1;
    int32_t alloc_off = 0;             // descriptor region allocator (pbuf2 / sstk)
    std::vector<PartDesc> small2;      // small parts cut from giant parts
    std::vector<GiantRec> giants;
    int64_t unresolved = 0, splits = 0;
    bool changed = false;
    int32_t *pbuf2 = nullptr, *psz = nullptr;
};

// process one giant part (members: order[lo..hi) with gmark == pid), recursively
int64_t giant_process(PosCtx &P, int64_t cbase, int64_t lo, int64_t hi, int32_t pid,
                      int32_t root) {
    slm_ctx *ctx = P.ctx;
    cudaStream_t s = ctx->stream;
    GiantArgs &A = P.GA;
    const int64_t N = hi - lo;
    const int64_t gid = (int64_t)P.giants.size();
    P.giants.emplace_back();
    // state
    GiantState h0;
    memset(&h0, 0, sizeof(h0));
    h0.pid = pid;
    h0.root = root;
    int32_t ar = 0, aq = 0;
    CUDA_TRY(cudaMemcpyAsync(&ar, A.a + root, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (ar != root) {
        CUDA_TRY(cudaMemcpyAsync(&aq, A.a + ar, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        SLM_REQUIRE(aq == root, SLM_EUNSUP, "assignment cycle longer than 2 in POSITIVE");
        h0.q = ar;
        h0.two = 1;
    } else {
        h0.q = root;
        h0.two = 0;
    }
    CUDA_TRY(cudaMemcpyAsync(P.S.p, &h0, sizeof(h0), cudaMemcpyHostToDevice, s));
    // full pass: w_part, LCA deposits, subtree sums
    unsigned GW = grid_for(N * 32, 256, 148LL * 32);
    unsigned GN = grid_for(N, 256);
    k_g_wpart<<<GW, 256, 0, s>>>(A, lo, hi, pid);
    k_g_lca<<<GW, 256, 0, s>>>(A, lo, hi, pid);
    P.vso.resize(N + 1);
    P.vsi.resize(N + 1);
    P.vdp.resize(N + 1);
    P.pso.resize(N + 1);
    P.psi.resize(N + 1);
    P.pdp.resize(N + 1);
    k_g_gather<<<GN, 256, 0, s>>>(A, lo, hi, pid, P.vso.p, P.vsi.p, P.vdp.p);
    CUDA_TRY(cudaMemsetAsync(P.vso.p + N, 0, 8, s));
    CUDA_TRY(cudaMemsetAsync(P.vsi.p + N, 0, 8, s));
    CUDA_TRY(cudaMemsetAsync(P.vdp.p + N, 0, 8, s));
    {
        size_t tb = 0;
        CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, P.vso.p, P.pso.p, N + 1, s));
        ctx->tmp.resize(tb);
        CUDA_TRY(cub::DeviceScan::ExclusiveSum(ctx->tmp.p, tb, P.vso.p, P.pso.p, N + 1, s));
        CUDA_TRY(cub::DeviceScan::ExclusiveSum(ctx->tmp.p, tb, P.vsi.p, P.psi.p, N + 1, s));
        CUDA_TRY(cub::DeviceScan::ExclusiveSum(ctx->tmp.p, tb, P.vdp.p, P.pdp.p, N + 1, s));
    }
    k_g_subsums<<<GN, 256, 0, s>>>(A, lo, hi, cbase, pid, P.pso.p, P.psi.p, P.pdp.p, P.S.p);
    // split loop
    const unsigned GE = std::min<unsigned>(GN, 148 * 8);
    P.blk_neg.resize(GE);
    P.blk_g.resize(GE);
    P.blk_x.resize(GE);
    int64_t neg_left = 0;
    for (;;) {
        k_g_eval<<<GE, GE_BLOCK, 0, s>>>(A, lo, hi, P.S.p, P.blk_neg.p, P.blk_g.p, P.blk_x.p);
        k_g_reduce<<<1, 32, 0, s>>>(A, GE, P.blk_neg.p, P.blk_g.p, P.blk_x.p, P.S.p);
        GiantState h;
        CUDA_TRY(cudaMemcpyAsync(&h, P.S.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        if (h.neg == 0) break;
        int32_t xc = -1;
        int pair = 0;
        double gain = 0.0;
        if (h.best_x != 0x7fffffff && h.best_gain > 0.0) {
            xc = h.best_x;
            gain = h.best_gain;
        } else if (h.two && h.pair_gain > 0.0) {
            xc = h.q;
            pair = 1;
            gain = h.pair_gain;
        }
        if (xc < 0) {
            neg_left = h.neg;
            break;
        }
        int32_t xpar = 0;
        CUDA_TRY(cudaMemcpyAsync(&xpar, A.a + xc, 4, cudaMemcpyDeviceToHost, s));
        const int32_t pid_b = P.next_pid++;
        CUDA_TRY(cudaMemsetAsync(&P.S.p->bsize, 0, 4, s));
        int32_t pxc = 0, sxc = 0;
        CUDA_TRY(cudaMemcpyAsync(&pxc, A.pos + xc, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(&sxc, A.sz + xc, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        const int64_t blo = cbase + pxc, bhi = blo + sxc;
        k_g_cut_mark<<<grid_for(sxc, 256), 256, 0, s>>>(A, cbase, xc, pid, pid_b, P.S.p);
        k_g_apply<<<1, 32, 0, s>>>(A, xc, pair, P.S.p);
        k_g_cross<<<grid_for((int64_t)sxc * 32, 256, 148LL * 32), 256, 0, s>>>(A, cbase, xc, xpar,
                                                                              pid, pid_b);
        int32_t bsize = 0;
        CUDA_TRY(cudaMemcpyAsync(&bsize, &P.S.p->bsize, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        P.changed = true;
        P.splits++;
        Split sp;
        sp.gain = gain;
        if (bsize <= SMALL_PART) {
            // compact b into its own region for the warp executor
            const int32_t off = P.alloc_off;
            P.alloc_off += bsize;
            const int64_t L = bhi - blo;
            P.cflag.resize(L + 1);
            P.cidx.resize(L + 1);
            DBuf<int32_t> posb;
            posb.resize(bsize);
            k_g_compact_flags<<<grid_for(L, 256), 256, 0, s>>>(A.order, A.gmark, blo, bhi, pid_b,
                                                               P.cflag.p);
            CUDA_TRY(cudaMemsetAsync(P.cflag.p + L, 0, 4, s));
            cub_exclusive_sum<int32_t>(ctx, P.cflag.p, P.cidx.p, L + 1);
            k_g_compact_fill<<<grid_for(L, 256), 256, 0, s>>>(A.order, A.pos, P.cflag.p,
                                                              P.cidx.p, blo, bhi, off, P.pbuf2,
                                                              posb.p);
            k_g_compact_psz<<<grid_for(bsize, 256), 256, 0, s>>>(P.pbuf2, posb.p, A.sz, off,
                                                                 bsize, P.psz);
            CUDA_TRY(cudaStreamSynchronize(s));
            PartDesc d;
            d.off = off;
            d.len = bsize;
            d.from_layout = 0;
            d.pad = 0;
            sp.kind = 0;
            sp.child = (int64_t)P.small2.size();
            P.small2.push_back(d);
        } else {
            GiantState saved;
            CUDA_TRY(cudaMemcpyAsync(&saved, P.S.p, sizeof(saved), cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            sp.kind = 1;
            sp.child = giant_process(P, cbase, blo, bhi, pid_b, xc);
            CUDA_TRY(cudaMemcpyAsync(P.S.p, &saved, sizeof(saved), cudaMemcpyHostToDevice, s));
            // the child used the shared scratch: recompute this part's block buffers lazily
            P.blk_neg.resize(GE);
            P.blk_g.resize(GE);
            P.blk_x.resize(GE);
        }
        P.giants[gid].splits.push_back(sp);
    }
    P.unresolved += neg_left;
    return gid;
}

void append_giant_gains(const PosCtx &P, int64_t gid, const std::vector<std::vector<double>> &sg,
                        std::vector<double> &out) {
    for (const Split &sp : P.giants[gid].splits) {
        out.push_back(sp.gain);
        if (sp.kind == 0) out.insert(out.end(), sg[sp.child].begin(), sg[sp.child].end());
        else append_giant_gains(P, sp.child, sg, out);
    }
}

}  // namespace

static void launch_small(slm_ctx *ctx, PosArgs &A, const std::vector<PartDesc> &parts,
                         DBuf<PartDesc> &dparts, DBuf<int32_t> &ngains, DBuf<int32_t> &nunres,
                         std::vector<int32_t> &hng, std::vector<int32_t> &hun) {
    cudaStream_t s = ctx->stream;
    const int64_t np = (int64_t)parts.size();
    hng.assign(np, 0);
    hun.assign(np, 0);
    if (np == 0) return;
    dparts.resize(np);
    ngains.resize(np);
    nunres.resize(np);
    CUDA_TRY(cudaMemcpyAsync(dparts.p, parts.data(), np * sizeof(PartDesc), cudaMemcpyHostToDevice, s));
    A.parts = dparts.p;
    A.nparts = np;
    A.ngains = ngains.p;
    A.neg_unres = nunres.p;
    k_positive<<<grid_for(np * 32, 128, 148LL * 64), 128, 0, s>>>(A);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(hng.data(), ngains.p, np * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(hun.data(), nunres.p, np * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
}

void run_positive(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m, int64_t scc_cap,
                  int64_t *splits, int64_t *unresolved, int *changed, std::vector<double> *gains) {
    (void)scc_cap;   // the scc_cut_cap branch needs cycles > cap >= 2: unreachable (F5)
    cudaStream_t s = ctx->stream;
    const int64_t n = G.n, nc = F.n_comms;
    *splits = 0;
    *unresolved = 0;
    *changed = 0;
    if (gains) gains->clear();
    if (m == 0.0 || n == 0) return;
    read_small_part();
    phase_mark(ctx, -1);
    DBuf<uint8_t> bad;
    bad.resize(nc);
    CUDA_TRY(cudaMemsetAsync(bad.p, 0, nc, s));
    run_local_gains(ctx, G, F, m, nullptr, bad.p);
    DBuf<int32_t> f, pos, list;
    f.resize(nc + 1);
    pos.resize(nc + 1);
    CUDA_TRY(cudaMemsetAsync(f.p + nc, 0, 4, s));
    k_bad_flags<<<grid_for(nc, 256), 256, 0, s>>>(bad.p, nc, f.p);
    cub_exclusive_sum<int32_t>(ctx, f.p, pos.p, nc + 1);
    int32_t nbad = 0;
    CUDA_TRY(cudaMemcpyAsync(&nbad, pos.p + nc, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (nbad == 0) return;
    list.resize(nbad);
    k_bad_scatter<<<grid_for(nc, 256), 256, 0, s>>>(f.p, pos.p, nc, list.p);
    phase_mark(ctx, PH_POS_LG);
    std::vector<int32_t> hbad(nbad), hcptr(nc + 1);
    CUDA_TRY(cudaMemcpyAsync(hbad.data(), list.p, nbad * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(hcptr.data(), F.cptr.p, (nc + 1) * 4, cudaMemcpyDeviceToHost, s));
    if (g_stamp.p == nullptr) {
        g_stamp.resize(1);
        CUDA_TRY(cudaMemsetAsync(g_stamp.p, 0, 4, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    // scratch (n-sized)
    DBuf<int32_t> pbuf, pbuf2, tbuf, pmark, ppos, psz, gmark, flags;
    DBuf<int2> sstk, sstk2;
    DBuf<double> wpart, dep, pso, psi, pdp, gbuf, gbuf2, xw, sob, sib;
    pbuf.resize(n); pbuf2.resize(n); tbuf.resize(n); pmark.resize(n); ppos.resize(n);
    psz.resize(n); gmark.resize(n); sstk.resize(n); sstk2.resize(n);
    wpart.resize(n); dep.resize(n); pso.resize(n); psi.resize(n); pdp.resize(n);
    gbuf.resize(n); gbuf2.resize(n);
    flags.resize(2);
    CUDA_TRY(cudaMemsetAsync(pmark.p, 0, n * 4, s));
    CUDA_TRY(cudaMemsetAsync(flags.p, 0, 8, s));
    PosArgs A;
    A.uptr = G.uptr.p;
    A.unbr = G.unbr.p;
    A.uu = G.uu.p;
    A.s_out = G.s_out.p;
    A.s_in = G.s_in.p;
    A.a = F.a.p;
    A.order = F.order.p;
    A.sz0 = F.sz.p;
    A.m = m;
    A.m2 = m * m;
    A.pbuf = pbuf.p;
    A.tbuf = tbuf.p;
    A.pmark = pmark.p;
    A.ppos = ppos.p;
    A.psz = psz.p;
    A.sstk = sstk.p;
    A.wpart = wpart.p;
    A.dep = dep.p;
    A.pre_so = pso.p;
    A.pre_si = psi.p;
    A.pre_dep = pdp.p;
    A.gains = gbuf.p;
    A.stamp_ctr = g_stamp.p;
    A.flags = flags.p;
    // 1. small bad communities straight from the layout
    std::vector<PartDesc> small1;
    std::vector<int64_t> order_kind(nbad);   // >=0: small1 index, <0: -(giant id)-1
    std::vector<int64_t> giant_of;
    std::vector<int32_t> giant_comm;
    for (int32_t i = 0; i < nbad; i++) {
        int32_t c = hbad[i];
        int32_t sz = hcptr[c + 1] - hcptr[c];
        if (sz <= SMALL_PART) {
            PartDesc d;
            d.off = hcptr[c];
            d.len = sz;
            d.from_layout = 1;
            d.pad = 0;
            order_kind[i] = (int64_t)small1.size();
            small1.push_back(d);
        } else {
            order_kind[i] = -1 - (int64_t)giant_comm.size();
            giant_comm.push_back(c);
        }
    }
    DBuf<PartDesc> dparts;
    DBuf<int32_t> ngains, nunres;
    std::vector<int32_t> hng1, hun1, hng2, hun2;
    launch_small(ctx, A, small1, dparts, ngains, nunres, hng1, hun1);
    phase_mark(ctx, PH_POS_SMALL);
    int64_t tot = 0, un = 0;
    for (size_t i = 0; i < small1.size(); i++) {
        tot += hng1[i];
        un += hun1[i];
    }
    // 2. giant communities: incremental grid executor; small cut subtrees -> batch 2
    PosCtx P;
    P.ctx = ctx;
    P.G = &G;
    P.F = &F;
    P.m = m;
    P.S.resize(1);
    P.pbuf2 = pbuf2.p;
    P.psz = psz.p;
    std::vector<int64_t> giant_ids;
    if (!giant_comm.empty()) {
        xw.resize(n);
        sob.resize(n);
        sib.resize(n);
        GiantArgs &GA = P.GA;
        GA.uptr = G.uptr.p;
        GA.unbr = G.unbr.p;
        GA.uu = G.uu.p;
        GA.s_out = G.s_out.p;
        GA.s_in = G.s_in.p;
        GA.a = F.a.p;
        GA.order = F.order.p;
        GA.pos = F.pos.p;
        GA.sz = F.sz.p;
        GA.gmark = gmark.p;
        GA.wpart = wpart.p;
        GA.dep = dep.p;
        GA.xw = xw.p;
        GA.sob = sob.p;
        GA.sib = sib.p;
        GA.m = m;
        GA.m2 = m * m;
        k_init_i32<<<grid_for(n, 256), 256, 0, s>>>(gmark.p, n, 0);
        for (int32_t c : giant_comm) {
            const int64_t lo = hcptr[c], hi = hcptr[c + 1];
            const int32_t pid = P.next_pid++;
            k_g_mark<<<grid_for(hi - lo, 256), 256, 0, s>>>(F.order.p, lo, hi, pid, gmark.p);
            int32_t root = 0;
            CUDA_TRY(cudaMemcpyAsync(&root, F.order.p + lo, 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            giant_ids.push_back(giant_process(P, lo, lo, hi, pid, root));
        }
        tot += P.splits;
        un += P.unresolved;
        // small parts cut from giants (their own regions in pbuf2 / sstk2 / gbuf2)
        A.pbuf = pbuf2.p;
        A.sstk = sstk2.p;
        A.gains = gbuf2.p;
        launch_small(ctx, A, P.small2, dparts, ngains, nunres, hng2, hun2);
        for (size_t i = 0; i < P.small2.size(); i++) {
            tot += hng2[i];
            un += hun2[i];
        }
    }
    int32_t hflags[2];
    CUDA_TRY(cudaMemcpyAsync(hflags, flags.p, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    phase_mark(ctx, PH_POS_GIANT);
    SLM_REQUIRE(!hflags[1], SLM_EUNSUP, "assignment cycle longer than 2 in POSITIVE");
    *splits = tot;
    *unresolved = un;
    *changed = hflags[0] || P.changed;
    if (gains && tot > 0) {
        // the reference's order: communities ascending; within a community its LIFO stack,
        // i.e. a cut's gain, then the cut subtree's gains, then the rest's
        std::vector<double> hg1(n), hg2(n);
        CUDA_TRY(cudaMemcpyAsync(hg1.data(), gbuf.p, n * 8, cudaMemcpyDeviceToHost, s));
        if (!P.small2.empty())
            CUDA_TRY(cudaMemcpyAsync(hg2.data(), gbuf2.p, n * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        std::vector<std::vector<double>> sg2(P.small2.size());
        for (size_t i = 0; i < P.small2.size(); i++)
            sg2[i].assign(hg2.begin() + P.small2[i].off, hg2.begin() + P.small2[i].off + hng2[i]);
        for (int32_t i = 0; i < nbad; i++) {
            if (order_kind[i] >= 0) {
                const PartDesc &d = small1[order_kind[i]];
                for (int k = 0; k < hng1[order_kind[i]]; k++) gains->push_back(hg1[d.off + k]);
            } else {
                append_giant_gains(P, giant_ids[-1 - order_kind[i]], sg2, *gains);
            }
        }
    }
}
