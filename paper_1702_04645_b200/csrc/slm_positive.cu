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
#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <functional>
#include <map>

// parts up to this size use the warp executor; SLM_SMALL_PART overrides it (tests force the
// giant executor onto small graphs with it)
static int SMALL_PART = 4096;
// members whose union rows exceed HEAVY_DEG entries send their community to the CTA executor
// (SLM_HEAVY_DEG overrides it; read with SLM_SMALL_PART at every call, cached per level graph)
static int64_t HEAVY_DEG = 1 << 16;
static void read_small_part() {
    const char *e = getenv("SLM_SMALL_PART");
    SMALL_PART = e ? std::max(1, atoi(e)) : 4096;
    const char *h = getenv("SLM_HEAVY_DEG");
    HEAVY_DEG = h ? std::max<int64_t>(1, atoll(h)) : (1 << 16);
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
            // LCA deposits: -u at the lowest ancestor of y whose DFS range holds z (lanes over
            // the entries of one member at a time: coarse-level rows can be long)
            auto deposit = [&](int32_t y, int64_t e) {
                const int32_t z = A.unbr[e];
                if (A.pmark[z] != (int32_t)stamp) return;
                const int32_t pz = A.ppos[z];
                int32_t anc = y;
                for (;;) {
                    const int32_t pa = A.ppos[anc];
                    if (pz >= pa && pz < pa + A.psz[anc]) break;
                    anc = A.a[anc];
                }
                atomicAdd(&A.dep[anc], -A.uu[e]);
            };
            for (int cb = 0; cb < len; cb += 32) {
                const int k = cb + lane;
                bool longrow = false;
                if (k < len) {
                    const int32_t y = P[k];
                    const int64_t e0 = A.uptr[y], e1 = A.uptr[y + 1];
                    if (e1 - e0 > 32) longrow = true;
                    else
                        for (int64_t e = e0; e < e1; e++) deposit(y, e);
                }
                unsigned lm = __ballot_sync(0xffffffffu, longrow);
                while (lm) {   // long rows: lanes over the entries
                    const int src = __ffs(lm) - 1;
                    lm &= lm - 1;
                    const int32_t y = P[cb + src];
                    for (int64_t e = A.uptr[y] + lane; e < A.uptr[y + 1]; e += 32) deposit(y, e);
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
    double *accl;            // per-node deposit scratch of the cut update (kept zero)
    // intra-part adjacency of the wave-0 parts (a superset for every descendant part):
    // node x's entries to members of its part are (iz, iu)[ioff[x], ioff[x] + icnt[x])
    int64_t *ioff;
    int32_t *icnt;
    int32_t *iz;
    double *iu;
    int32_t *iy;             // owner of each entry (the flat LCA pass of wave 0)
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
    if (S && blockIdx.x == 0 && threadIdx.x == 0) {
        S->so_c = pso[hi - lo];
        S->si_c = psi[hi - lo];
    }
}

__global__ void k_bad_flags(const uint8_t *bad, int64_t nc, int32_t *f) {
    GS_LOOP(c, nc) f[c] = bad[c] ? 1 : 0;
}
__global__ void k_bad_scatter(const int32_t *f, const int32_t *pos, int64_t nc, int32_t *list) {
    GS_LOOP(c, nc) if (f[c]) list[pos[c]] = (int32_t)c;
}
__global__ void k_init_i32(int32_t *x, int64_t n, int32_t v) { GS_LOOP(i, n) x[i] = v; }
__global__ void k_bad_ranges(const int32_t *list, int64_t nbad, const int32_t *cptr, int2 *out) {
    GS_LOOP(i, nbad) out[i] = make_int2(cptr[list[i]], cptr[list[i] + 1]);
}
// members whose rows exceed HEAVY_DEG entries mark their community "heavy": a warp rescans
// every member row at each split, so such parts go to the CTA executor instead
__global__ void k_heavy_flags(const int64_t *uptr, int64_t n, int64_t heavy_deg, int32_t *f) {
    GS_LOOP(i, n) f[i] = uptr[i + 1] - uptr[i] > heavy_deg ? 1 : 0;
}
__global__ void k_heavy_scatter(const int32_t *f, const int32_t *pos, int64_t n, int32_t *out) {
    GS_LOOP(i, n) if (f[i]) out[pos[i]] = (int32_t)i;
}
__global__ void k_heavy_mark(const int32_t *nodes, int64_t k, const int32_t *comm, uint8_t *heavy) {
    GS_LOOP(i, k) heavy[comm[nodes[i]]] = 1;
}
__global__ void k_bad_heavy(const int32_t *list, int64_t nbad, const uint8_t *heavy, uint8_t *out) {
    GS_LOOP(i, nbad) out[i] = heavy[list[i]];
}

// ---- batched init of every part of a giant wave.  Parts are slices [lo, hi) of the layout
// (members: gmark == pid); their concatenation is indexed by a flat index t.  Member rows are
// cut into chunks of GCH entries (one warp per chunk), so hub members do not serialise a warp.
constexpr int GCH = 1024;
struct GSlice {
    int64_t lo, hi, cbase, flat;   // flat: start of the slice in the concatenation
    int32_t pid, pad;
};
__device__ __forceinline__ int slice_of(const GSlice *S, int ns, int64_t t) {
    int a = 0, b = ns - 1;
    while (a < b) {   // last slice with flat <= t
        const int mid = (a + b + 1) >> 1;
        if (S[mid].flat <= t) a = mid;
        else b = mid - 1;
    }
    return a;
}
__global__ void k_gb_chunks(GiantArgs A, const GSlice *S, int ns, int64_t N, int32_t *nch,
                            int build_intra) {
    GS_LOOP(t, N) {
        const GSlice sl = S[slice_of(S, ns, t)];
        const int32_t x = A.order[sl.lo + (t - sl.flat)];
        int32_t c = 0;
        if (A.gmark[x] == sl.pid) {
            const int64_t d = A.uptr[x + 1] - A.uptr[x];
            c = (int32_t)((d + GCH - 1) / GCH);
            A.wpart[x] = 0.0;
            if (build_intra) A.icnt[x] = 0;
        }
        nch[t] = c;
    }
}
__global__ void k_gb_expand(GiantArgs A, const GSlice *S, int ns, int64_t N, const int32_t *nch,
                            const int64_t *choff, int64_t *chunks) {
    GS_LOOP(t, N) {
        const int64_t o = choff[t];
        for (int32_t c = 0; c < nch[t]; c++) chunks[o + c] = (t << 22) | c;
    }
}
__device__ __forceinline__ int32_t chunk_node(const GiantArgs &A, const GSlice *S, int ns, int64_t ck,
                                              int64_t &e0, int64_t &e1) {
    const int64_t t = ck >> 22, c = ck & 0x3FFFFF;
    const GSlice sl = S[slice_of(S, ns, t)];
    const int32_t x = A.order[sl.lo + (t - sl.flat)];
    const int64_t b = A.uptr[x], d = A.uptr[x + 1] - b;
    e0 = b + c * GCH;
    e1 = b + min(d, (c + 1) * (int64_t)GCH);
    return x;
}
__global__ void k_gb_wpart(GiantArgs A, const GSlice *S, int ns, const int64_t *chunks, int64_t nck,
                           int build_intra) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = w; k < nck; k += nw) {
        int64_t e0, e1;
        const int32_t x = chunk_node(A, S, ns, chunks[k], e0, e1);
        const int32_t pid = A.gmark[x];
        double wp = 0.0;
        int ni = 0;
        for (int64_t e = e0 + lane; e < e1; e += 32)
            if (A.gmark[A.unbr[e]] == pid) {
                wp += A.uu[e];
                ni++;
            }
        wp = wsum_d(wp);
        ni = __reduce_add_sync(0xffffffffu, ni);
        if (lane == 0 && wp != 0.0) atomicAdd(&A.wpart[x], wp);
        if (build_intra && lane == 0 && ni) atomicAdd(&A.icnt[x], ni);
    }
}
__global__ void k_gb_icount(GiantArgs A, const GSlice *S, int ns, int64_t N, int64_t *cnt) {
    GS_LOOP(t, N) {
        const GSlice sl = S[slice_of(S, ns, t)];
        const int32_t x = A.order[sl.lo + (t - sl.flat)];
        cnt[t] = A.gmark[x] == sl.pid ? A.icnt[x] : 0;
    }
}
__global__ void k_gb_ioff(GiantArgs A, const GSlice *S, int ns, int64_t N, const int64_t *off) {
    GS_LOOP(t, N) {
        const GSlice sl = S[slice_of(S, ns, t)];
        const int32_t x = A.order[sl.lo + (t - sl.flat)];
        if (A.gmark[x] == sl.pid) {
            A.ioff[x] = off[t];
            A.icnt[x] = 0;   // refilled by k_gb_ifill
        }
    }
}
__global__ void k_gb_ifill(GiantArgs A, const GSlice *S, int ns, const int64_t *chunks, int64_t nck) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = w; k < nck; k += nw) {
        int64_t e0, e1;
        const int32_t x = chunk_node(A, S, ns, chunks[k], e0, e1);
        const int32_t pid = A.gmark[x];
        for (int64_t eb = e0; eb < e1; eb += 32) {
            const int64_t e = eb + lane;
            int32_t z = 0;
            bool hit = false;
            if (e < e1) {
                z = A.unbr[e];
                hit = A.gmark[z] == pid;
            }
            const unsigned hm = __ballot_sync(0xffffffffu, hit);
            if (!hm) continue;
            int at = 0;
            if (lane == 0) at = atomicAdd(&A.icnt[x], __popc(hm));
            at = __shfl_sync(0xffffffffu, at, 0);
            if (hit) {
                const int64_t q = A.ioff[x] + at + __popc(hm & ((1u << lane) - 1));
                A.iz[q] = z;
                A.iu[q] = A.uu[e];
                if (A.iy) A.iy[q] = x;
            }
        }
    }
}
__global__ void k_gb_dep(GiantArgs A, const GSlice *S, int ns, int64_t N) {
    GS_LOOP(t, N) {
        const GSlice sl = S[slice_of(S, ns, t)];
        const int32_t x = A.order[sl.lo + (t - sl.flat)];
        if (A.gmark[x] == sl.pid) A.dep[x] = A.wpart[x];
    }
}
__global__ void k_gb_lca(GiantArgs A, const GSlice *S, int ns, const int64_t *chunks, int64_t nck) {
    // over the intra-part lists (chunk c of a member covers its list range [c, c+1) * GCH;
    // the lists are never longer than the rows, so some chunks are empty)
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = w; k < nck; k += nw) {
        const int64_t t = chunks[k] >> 22, c = chunks[k] & 0x3FFFFF;
        const GSlice sl = S[slice_of(S, ns, t)];
        const int32_t y = A.order[sl.lo + (t - sl.flat)];
        const int32_t pid = A.gmark[y];
        const int64_t b0 = A.ioff[y], cnt = A.icnt[y];
        const int64_t q0 = b0 + c * GCH, q1 = b0 + min(cnt, (c + 1) * (int64_t)GCH);
        // y's ancestor chain is shared by the whole row: lane i holds level i (node and DFS
        // interval), extended one level at a time only as far as some lane's entry needs, so
        // every entry finds its LCA by shuffles; entries above 32 levels walk on from there.
        // Deposits are cached per lane while the LCA repeats (in a hub-centred tree most
        // edges meet at the root: one atomic per run instead of one per edge).
        int32_t ch_node = -1, ch_lo = 0, ch_hi = 0;
        int clen = 0;
        int32_t nxt = y;   // next node to append to the chain
        int32_t ca = -1;
        double cv = 0.0;
        for (int64_t qb = q0; qb < q1; qb += 32) {
            const int64_t q = qb + lane;
            bool need = false;
            int32_t pz = 0;
            double u = 0.0;
            if (q < q1) {
                const int32_t z = A.iz[q];
                u = A.iu[q];
                if (A.gmark[z] == pid) {
                    need = true;
                    pz = A.pos[z];
                }
            }
            int32_t anc = -1;
            for (int L = 0; L < clen; L++) {
                const int32_t lo = __shfl_sync(0xffffffffu, ch_lo, L);
                const int32_t hi = __shfl_sync(0xffffffffu, ch_hi, L);
                const int32_t nd = __shfl_sync(0xffffffffu, ch_node, L);
                if (need && anc < 0 && pz >= lo && pz < hi) anc = nd;
            }
            while (clen < 32 && __any_sync(0xffffffffu, need && anc < 0)) {
                const int32_t nd = nxt;   // uniform across the warp
                const int32_t pa = A.pos[nd], sa = A.sz[nd], an = A.a[nd];
                if (lane == clen) {
                    ch_node = nd;
                    ch_lo = pa;
                    ch_hi = pa + sa;
                }
                clen++;
                nxt = an;
                if (need && anc < 0 && pz >= pa && pz < pa + sa) anc = nd;
            }
            if (need && anc < 0) {   // deeper than 32 levels: walk on from the chain's end
                int32_t w2 = nxt;
                for (;;) {
                    const int32_t pa = A.pos[w2], sa = A.sz[w2], an = A.a[w2];
                    if (pz >= pa && pz < pa + sa) break;
                    w2 = an;
                }
                anc = w2;
            }
            if (need) {
                if (anc != ca) {
                    if (ca >= 0) atomicAdd(&A.dep[ca], cv);
                    ca = anc;
                    cv = 0.0;
                }
                cv -= u;
            }
        }
        if (ca >= 0) atomicAdd(&A.dep[ca], cv);
    }
}
// wave 0: one thread per intra-list entry (the lists are short, so a warp per member row
// leaves most lanes idle).  The owner y walks up to the lowest ancestor whose DFS interval
// holds z; runs of equal ancestors across the warp's lanes share one atomic.
__global__ void k_gb_lca_flat(GiantArgs A, int64_t nintra) {
    const int lane = threadIdx.x & 31;
    for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31LL; b < nintra;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = b + lane;
        int32_t anc = -1;
        double v = 0.0;
        if (q < nintra) {
            const int32_t y = A.iy[q], z = A.iz[q];
            const double u = A.iu[q];
            const int32_t gy = A.gmark[y], gz = A.gmark[z], pz = A.pos[z];
            if (gy == gz) {
                int32_t w = y;
                int32_t pa = A.pos[w], sa = A.sz[w], nx = A.a[w];
                while (!(pz >= pa && pz < pa + sa)) {
                    w = nx;
                    pa = A.pos[w];
                    sa = A.sz[w];
                    nx = A.a[w];
                }
                anc = w;
                v = -u;
            }
        }
        // segmented scan over runs of equal ancestors (a value may recur in later runs)
        const int32_t pa = __shfl_up_sync(0xffffffffu, anc, 1);
        const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || pa != anc);
        const int start = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double ov = __shfl_up_sync(0xffffffffu, v, off);
            if (lane - off >= start) v += ov;
        }
        const int32_t na = __shfl_down_sync(0xffffffffu, anc, 1);
        if (anc >= 0 && (lane == 31 || na != anc)) atomicAdd(&A.dep[anc], v);
    }
}

__global__ void k_gb_gather(GiantArgs A, const GSlice *S, int ns, int64_t N, double *vso,
                            double *vsi, double *vdp) {
    GS_LOOP(t, N) {
        const GSlice sl = S[slice_of(S, ns, t)];
        const int32_t x = A.order[sl.lo + (t - sl.flat)];
        const bool in = A.gmark[x] == sl.pid;
        vso[t] = in ? A.s_out[x] : 0.0;
        vsi[t] = in ? A.s_in[x] : 0.0;
        vdp[t] = in ? A.dep[x] : 0.0;
    }
}
__global__ void k_gb_subsums(GiantArgs A, const GSlice *S, int ns, int64_t N, const double *pso,
                             const double *psi, const double *pdp) {
    GS_LOOP(t, N) {
        const GSlice sl = S[slice_of(S, ns, t)];
        const int32_t x = A.order[sl.lo + (t - sl.flat)];
        if (A.gmark[x] != sl.pid) continue;
        const int64_t i0 = sl.flat + sl.cbase + A.pos[x] - sl.lo, i1 = i0 + A.sz[x];
        A.sob[x] = pso[i1] - pso[i0];
        A.sib[x] = psi[i1] - psi[i0];
        A.xw[x] = pdp[i1] - pdp[i0];
    }
}


// ------------------------------------------------ giant parts: one CTA per part

constexpr int GB = 1024;              // threads per giant-part CTA
constexpr int GT = 512;               // top candidate list kept between full passes
constexpr int GLOC = 4;               // per-thread candidates of a full pass
constexpr int GSORT = GB * GLOC;      // sorted in (dynamic) shared memory
constexpr size_t GSMEM = (size_t)GSORT * (sizeof(double) + sizeof(int32_t));
constexpr int DIRTY_CAP = 1 << 16;    // locally updated nodes before a forced full pass
constexpr int CHAIN_CAP = 2048;       // ancestor chain of a cut kept in shared memory
constexpr int BIG_ROW = 2048;         // cut-subtree members with longer rows: CTA-wide
constexpr int BIG_CAP = 256;

struct GPart {
    int64_t lo, hi, cbase;   // member slice (community DFS coordinates) and community base
    int32_t pid, root;
    double so_c, si_c;
    int64_t neg_off;         // region of hi-lo entries in the negative-member pool
    int64_t dirty_off;       // region of DIRTY_CAP entries in the dirty pool
};

__global__ void k_gb_totals(const GSlice *S, int ns, const double *pso, const double *psi,
                            GPart *P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < ns) {
        const GSlice sl = S[i];
        const int64_t a = sl.flat, b = sl.flat + (sl.hi - sl.lo);
        P[i].so_c = pso[b] - pso[a];
        P[i].si_c = psi[b] - psi[a];
    }
}

struct GOut {
    // split log: (part pid, sequence, gain, child kind 0 small / 1 giant, child id)
    int32_t *log_pid, *log_seq, *log_kind, *log_child;
    double *log_gain;
    int32_t *nlog;
    // small children: descriptors + compacted members (warp executor, second batch)
    PartDesc *desc;
    int32_t *ndesc;
    int32_t *pbuf2, *posb, *psz;
    int32_t *alloc;
    // giant children: next wave
    int64_t *nx_lo, *nx_hi;
    int32_t *nx_pid, *nx_root, *nx_size;
    int32_t *nnext;
    int32_t *pid_ctr;
    unsigned long long *unresolved;
    int32_t *flags;          // [0] changed, [1] unsupported cycle
    int32_t small_part;      // cut subtrees up to this size go to the warp executor
    unsigned long long *prof;   // SLM_POS_LOG section cycle counters (else nullptr)
};

__device__ __forceinline__ double g_member(const GiantArgs &A, int32_t x, double so_c, double si_c) {
    const double sox = A.s_out[x], six = A.s_in[x];
    return A.wpart[x] / A.m - (sox * (si_c - six) + six * (so_c - sox)) / A.m2;
}
__device__ __forceinline__ double g_branch(const GiantArgs &A, int32_t x, double so_c, double si_c) {
    const double so_b = A.sob[x], si_b = A.sib[x];
    const double null = -so_c * si_b - so_b * si_c + 2.0 * so_b * si_b;
    return -A.xw[x] / A.m - null / (A.m * A.m);
}
__device__ __forceinline__ bool gbetter(double g1, int32_t x1, double g2, int32_t x2) {
    return g1 > g2 || (g1 == g2 && x1 < x2);
}

// block argmax of (g desc, x asc); result valid in every thread
__device__ void block_best(double &g, int32_t &x, double *sg, int32_t *sx) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double og = __shfl_xor_sync(0xffffffffu, g, o);
        const int32_t ox = __shfl_xor_sync(0xffffffffu, x, o);
        if (gbetter(og, ox, g, x)) {
            g = og;
            x = ox;
        }
    }
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sg[wid] = g;
        sx[wid] = x;
    }
    __syncthreads();
    if (wid == 0) {
        g = lane < GB / 32 ? sg[lane] : -INFINITY;
        x = lane < GB / 32 ? sx[lane] : 0x7fffffff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double og = __shfl_xor_sync(0xffffffffu, g, o);
            const int32_t ox = __shfl_xor_sync(0xffffffffu, x, o);
            if (gbetter(og, ox, g, x)) {
                g = og;
                x = ox;
            }
        }
        if (lane == 0) {
            sg[0] = g;
            sx[0] = x;
        }
    }
    __syncthreads();
    g = sg[0];
    x = sx[0];
    __syncthreads();
}

__device__ int block_sum_i(int v, int *si) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) si[wid] = v;
    __syncthreads();
    if (wid == 0) {
        v = lane < GB / 32 ? si[lane] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) si[0] = v;
    }
    __syncthreads();
    v = si[0];
    __syncthreads();
    return v;
}

__device__ __forceinline__ void mark_dirty(int32_t y, uint8_t *gflag, int32_t *dirty, int *ndirty,
                                           int *overflow) {
    // byte flag with a CAS on its aligned word
    unsigned int *wp = (unsigned int *)(gflag + (y & ~3));
    const unsigned int bit = 1u << ((y & 3) * 8);
    const unsigned int old = atomicOr(wp, bit);
    if (!(old & bit)) {
        const int at = atomicAdd(ndirty, 1);
        if (at < DIRTY_CAP) {
            dirty[at] = y;
        } else {   // not listed: leave it unflagged (the overflow forces a full pass)
            atomicAnd(wp, ~bit);
            *overflow = 1;
        }
    }
}

// one CTA per giant part: the reference's repeated best single cut (detector.py:210-284)
// with incremental state.  Between full passes every non-dirty candidate's branch gain
// can only decrease (the part totals shrink; its own subtree sums and crossing weight are
// unchanged), and every non-dirty member's gain can only increase, so the top list plus the
// bound tau decide most splits exactly without rescanning the part.
__global__ void __launch_bounds__(GB) k_giant_cta(GiantArgs A, const GPart *parts, GOut O,
                                                  int32_t *neg_pool, int32_t *dirty_pool,
                                                  uint8_t *gflag, uint8_t *negflag) {
    extern __shared__ __align__(16) unsigned char g_dyn[];
    double *tg = (double *)g_dyn;
    int32_t *tx = (int32_t *)(g_dyn + (size_t)GSORT * sizeof(double));
    __shared__ double sg[32];
    __shared__ int32_t sxx[32];
    __shared__ int si[32];
    __shared__ int s_nneg, s_ndirty, s_overflow;
    __shared__ double s_tau, s_so, s_si;
    __shared__ int s_ntop, s_two, s_nadd, s_topfull;
    __shared__ int32_t s_chain[CHAIN_CAP];
    __shared__ int32_t s_big[BIG_CAP];
    __shared__ int s_nbig, s_nch;
    const GPart P = parts[blockIdx.x];
    const int tid = threadIdx.x;
    const int32_t pid = P.pid, r = P.root;
    int32_t *negl = neg_pool + P.neg_off;
    int32_t *dirty = dirty_pool + P.dirty_off;
    const int32_t q = A.a[r];
    if (tid == 0) {
        s_two = (q != r);
        if (q != r && A.a[q] != r) atomicOr(&O.flags[1], 1);
        s_so = P.so_c;
        s_si = P.si_c;
        s_nneg = 0;
        s_ndirty = 0;
        s_overflow = 0;
        s_ntop = 0;
        s_nadd = 0;
        s_topfull = 0;
    }
    __syncthreads();
    if (s_two && A.a[q] != r) return;
    bool need_full = true;
    int seq = 0;
    const long long t_cta = clock64();
    long long tsec = clock64();
    auto sec = [&](int k) {
        if (O.prof && tid == 0) {
            const long long t = clock64();
            atomicAdd(O.prof + k, (unsigned long long)(t - tsec));
            atomicAdd(O.prof + 8 + 8 * (int64_t)blockIdx.x + k, (unsigned long long)(t - tsec));
            tsec = t;
        }
    };
    for (;;) {
        double so_c = s_so, si_c = s_si;
        const bool two = s_two;
        double bg = -INFINITY;
        int32_t bx = 0x7fffffff;
        int negc = 0;
        if (!need_full) {
            // incremental: re-evaluate the top list and the nodes the last cut touched.  A
            // touched node above the bound tau joins the top list (flag bit 1 keeps it there
            // once); the others are back under tau, so the touched list is cleared every cut
            const int ntop = s_ntop, nd = min(s_ndirty, DIRTY_CAP);
            const double tau = s_tau;
            for (int t = tid; t < ntop + nd; t += GB) {
                const int32_t x = t < ntop ? tx[t] : dirty[t - ntop];
                if (A.gmark[x] != pid || x == r || (two && x == q)) continue;
                const double g = g_branch(A, x, so_c, si_c);
                if (gbetter(g, x, bg, bx)) {
                    bg = g;
                    bx = x;
                }
                if (t >= ntop && g > tau) {
                    unsigned int *wp = (unsigned int *)(gflag + (x & ~3));
                    const unsigned int tb = 2u << ((x & 3) * 8);
                    if (!(atomicOr(wp, tb) & tb)) {
                        const int at = ntop + atomicAdd(&s_nadd, 1);
                        if (at < GSORT) {
                            tx[at] = x;
                        } else {
                            atomicAnd(wp, ~tb);
                            s_topfull = 1;
                        }
                    }
                }
            }
            block_best(bg, bx, sg, sxx);
            if (tid == 0) {
                s_ntop = min(ntop + s_nadd, GSORT);
                s_nadd = 0;
            }
            if (!(bg > tau) || s_overflow || s_topfull) need_full = true;
            sec(0);
        }
        if (need_full) {
            if (tid == 0) {
                atomicAdd(O.unresolved + 1, 1ull);
                atomicAdd(O.unresolved + 2, (unsigned long long)(P.hi - P.lo));
            }
            // reset the incremental state
            __syncthreads();
            for (int t = tid; t < min(s_ndirty, DIRTY_CAP); t += GB) gflag[dirty[t]] = 0;
            for (int t = tid; t < s_ntop; t += GB) gflag[tx[t]] = 0;
            for (int t = tid; t < s_nneg; t += GB) negflag[negl[t]] = 0;
            __syncthreads();
            if (tid == 0) {
                s_ndirty = 0;
                s_overflow = 0;
                s_nneg = 0;
                s_ntop = 0;
                s_nadd = 0;
                s_topfull = 0;
            }
            __syncthreads();
            double lg[GLOC];
            int32_t lx[GLOC];
#pragma unroll
            for (int u = 0; u < GLOC; u++) {
                lg[u] = -INFINITY;
                lx[u] = 0x7fffffff;
            }
            double drop = -INFINITY;
            // four strided members per step: their loads are issued together (the list is
            // order-independent: (gain desc, id asc) top list, max of the dropped gains)
            constexpr int FU = 4;
            for (int64_t k0 = P.lo + tid; k0 < P.hi; k0 += (int64_t)FU * GB) {
                int32_t xs[FU];
                bool ok[FU];
                double gmv[FU], gbv[FU];
#pragma unroll
                for (int u = 0; u < FU; u++) {
                    const int64_t kk = k0 + (int64_t)u * GB;
                    xs[u] = kk < P.hi ? A.order[kk] : -1;
                }
#pragma unroll
                for (int u = 0; u < FU; u++) ok[u] = xs[u] >= 0 && A.gmark[xs[u]] == pid;
#pragma unroll
                for (int u = 0; u < FU; u++) {
                    gmv[u] = ok[u] ? g_member(A, xs[u], so_c, si_c) : 0.0;
                    gbv[u] = ok[u] ? g_branch(A, xs[u], so_c, si_c) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < FU; u++) {
                const int32_t x = xs[u];
                if (!ok[u]) continue;
                if (gmv[u] < 0.0) {
                    negl[atomicAdd(&s_nneg, 1)] = x;
                    negflag[x] = 1;
                }
                if (x == r || (two && x == q)) continue;
                double g = gbv[u];
                int32_t xx = x;
#pragma unroll
                for (int u = 0; u < GLOC; u++) {   // insertion into the local top list
                    if (gbetter(g, xx, lg[u], lx[u])) {
                        const double tgv = lg[u];
                        const int32_t txv = lx[u];
                        lg[u] = g;
                        lx[u] = xx;
                        g = tgv;
                        xx = txv;
                    }
                }
                drop = fmax(drop, g);   // best candidate not kept locally
                }
            }
#pragma unroll
            for (int u = 0; u < GLOC; u++) {
                tg[tid * GLOC + u] = lg[u];
                tx[tid * GLOC + u] = lx[u];
            }
            // bitonic sort of the GSORT candidates, best first
            for (int kk = 2; kk <= GSORT; kk <<= 1) {
                for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                    __syncthreads();
                    for (int idx = tid; idx < GSORT; idx += GB) {
                        const int ixj = idx ^ jj;
                        if (ixj > idx) {
                            const bool up = (idx & kk) == 0;
                            const bool swap = up ? gbetter(tg[ixj], tx[ixj], tg[idx], tx[idx])
                                                 : gbetter(tg[idx], tx[idx], tg[ixj], tx[ixj]);
                            if (swap) {
                                const double a1 = tg[idx];
                                tg[idx] = tg[ixj];
                                tg[ixj] = a1;
                                const int32_t b1 = tx[idx];
                                tx[idx] = tx[ixj];
                                tx[ixj] = b1;
                            }
                        }
                    }
                }
            }
            __syncthreads();
            // tau: best candidate outside the kept list
            double dmax = drop;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
            if ((tid & 31) == 0) sg[tid >> 5] = dmax;
            __syncthreads();
            if (tid == 0) {
                double t = tg[GT];
                for (int w = 0; w < GB / 32; w++) t = fmax(t, sg[w]);
                s_tau = t;
                int nt = 0;
                while (nt < GT && tx[nt] != 0x7fffffff) nt++;
                s_ntop = nt;
            }
            __syncthreads();
            for (int t = tid; t < s_ntop; t += GB) gflag[tx[t]] = 2;   // in the top list
            bg = tg[0];
            bx = tx[0];
            need_full = false;
            sec(1);
        }
        // negative members: the previous ones plus the dirty ones.  Only the dirty members (a
        // cut lowered their w_part) can turn negative -- every other member's gain grows as
        // the part shrinks -- so they are added to the list; whether any negative member is
        // left is then decided by scanning the list only up to the first one still negative,
        // and the exact count is taken only when no positive cut remains (detector.py:275-277)
        {
            const int nd = min(s_ndirty, DIRTY_CAP);
            int c = 0;
            for (int t = tid; t < nd; t += GB) {
                const int32_t x = dirty[t];
                if (A.gmark[x] == pid && !negflag[x] && g_member(A, x, so_c, si_c) < 0.0) {
                    c++;
                    negflag[x] = 1;
                    negl[atomicAdd(&s_nneg, 1)] = x;
                }
            }
            __syncthreads();
            const int nn = s_nneg;
            int any = __syncthreads_or(c);
            for (int base = 0; !any && base < nn; base += GB) {
                const int t = base + tid;
                bool neg = false;
                if (t < nn) {
                    const int32_t x = negl[t];
                    neg = A.gmark[x] == pid && g_member(A, x, so_c, si_c) < 0.0;
                }
                any = __syncthreads_or(neg);
            }
            negc = any ? -1 : 0;   // -1: some negative member (count taken when needed)
            sec(2);
        }
        if (negc == 0) break;   // no member with negative gain left (detector.py:224-225)
        int32_t xc = -1;
        int pair = 0;
        double gain = 0.0;
        if (bx != 0x7fffffff && bg > 0.0) {
            xc = bx;
            gain = bg;
        } else if (two) {
            const double pg = [&] {   // pair cut (detector.py:254-274, 288-335 with s = 2)
                const double so_b = A.sob[q], si_b = A.sib[q];
                const double null = -so_c * si_b - so_b * si_c + 2.0 * so_b * si_b;
                return -A.xw[q] / A.m - null / A.m2;
            }();
            if (pg > 0.0) {
                xc = q;
                pair = 1;
                gain = pg;
            }
        }
        if (xc < 0) {   // the exact number of negative members (detector.py:275-277)
            const int nn = s_nneg;
            int c = 0;
            for (int t = tid; t < nn; t += GB) {
                const int32_t x = negl[t];
                if (A.gmark[x] == pid && g_member(A, x, so_c, si_c) < 0.0) c++;
            }
            negc = block_sum_i(c, si);
            if (tid == 0) atomicAdd(O.unresolved, (unsigned long long)negc);
            break;
        }
        // the touched nodes are consumed: clear their flags (keeping the top-list bit)
        {
            const int nd = min(s_ndirty, DIRTY_CAP);
            for (int t = tid; t < nd; t += GB) {
                const int32_t y = dirty[t];
                gflag[y] = __ldcg(gflag + y) & 2;
            }
            __syncthreads();
            if (tid == 0) s_ndirty = 0;
        }
        // ---- apply the cut: a, part totals, ancestors' subtree sums
        const int32_t xpar = A.a[xc];
        const double sb = A.sob[xc], ib = A.sib[xc];
        const int64_t blo = P.cbase + A.pos[xc], bhi = blo + A.sz[xc];
        int32_t pid_b = 0;
        __syncthreads();   // everyone has read a[xc] before it changes
        if (tid == 0) {
            pid_b = atomicAdd(O.pid_ctr, 1);
            sxx[0] = pid_b;
            s_so = so_c - sb;
            s_si = si_c - ib;
            O.flags[0] = 1;
            if (pair) {
                A.sob[r] -= sb;
                A.sib[r] -= ib;
                mark_dirty(r, gflag, dirty, &s_ndirty, &s_overflow);
                A.a[r] = r;
                A.a[xc] = xc;
                s_two = 0;
            } else {
                // the ancestor chain xpar .. r (parents only: the loop carries one dependent
                // load per step); the subtree-sum updates run CTA-wide below
                A.a[xc] = xc;
                int nch = 0;
                for (int32_t y = xpar;; y = A.a[y]) {
                    if (nch < CHAIN_CAP) s_chain[nch] = y;
                    nch++;
                    if (y == r) break;
                }
                s_nch = nch;
            }
        }
        __syncthreads();
        pid_b = sxx[0];
        if (!pair) {
            const int nch = s_nch;
            if (nch <= CHAIN_CAP) {
                for (int c = tid; c < nch; c += GB) {
                    const int32_t y = s_chain[c];
                    A.sob[y] -= sb;
                    A.sib[y] -= ib;
                    mark_dirty(y, gflag, dirty, &s_ndirty, &s_overflow);
                }
            } else if (tid == 0) {
                for (int32_t y = xpar;; y = A.a[y]) {
                    A.sob[y] -= sb;
                    A.sib[y] -= ib;
                    mark_dirty(y, gflag, dirty, &s_ndirty, &s_overflow);
                    if (y == r) break;
                }
            }
        }
        // re-mark the cut subtree
        int cb = 0;
        for (int64_t k = blo + tid; k < bhi; k += GB) {
            const int32_t x = A.order[k];
            if (A.gmark[x] == pid) {
                A.gmark[x] = pid_b;
                cb++;
            }
        }
        const int bsize = block_sum_i(cb, si);
        sec(3);
        // edges between b and the rest: w_part of the rest side, x_w along the tree paths.
        // Members with short rows: one warp each; long rows (hubs) afterwards with the
        // whole CTA, so a hub inside b does not serialise one warp.
        {
            const int lane = tid & 31, wid = tid >> 5;
            if (tid == 0) s_nbig = 0;
            __syncthreads();
            // (entries from the wave-0 intra-part lists: a superset of the part's edges)
            auto edge = [&](int64_t q, int32_t pz) {
                const int32_t v = A.iz[q];
                const double u = A.iu[q];
                // one round trip per step: the parent, the DFS interval and the dirty byte of
                // the next node are loaded before this node's updates are issued (a stale 0
                // flag only costs the deduplicating atomic); v's own come with its part mark
                const int32_t gm = A.gmark[v];
                int32_t pa = A.pos[v], sa = A.sz[v], nx = A.a[v];
                uint8_t df = gflag[v];
                if (gm != pid) return;
                atomicAdd(&A.wpart[v], -u);
                if (!(df & 1)) mark_dirty(v, gflag, dirty, &s_ndirty, &s_overflow);
                df = 1;
                int32_t y = v;
                while (!(pz >= pa && pz < pa + sa)) {
                    const int32_t y2 = nx;
                    const int32_t pa2 = A.pos[y2], sa2 = A.sz[y2], nx2 = A.a[y2];
                    const uint8_t df2 = gflag[y2];
                    atomicAdd(&A.xw[y], -u);
                    if (!(df & 1)) mark_dirty(y, gflag, dirty, &s_ndirty, &s_overflow);
                    y = y2;
                    pa = pa2;
                    sa = sa2;
                    nx = nx2;
                    df = df2;
                }
                // b-side: every ancestor of b strictly below lca = y loses u; deposited
                // at the lca and applied in one walk of b's ancestor chain below
                atomicAdd(&A.accl[y], u);
            };
            for (int64_t k = blo + wid; k < bhi; k += GB / 32) {
                const int32_t z = A.order[k];
                if (A.gmark[z] != pid_b) continue;
                const int64_t e0 = A.ioff[z], e1 = e0 + A.icnt[z];
                if (e1 - e0 > BIG_ROW) {
                    int at = 0;
                    if (lane == 0) {
                        at = atomicAdd(&s_nbig, 1);
                        if (at < BIG_CAP) s_big[at] = z;
                    }
                    at = __shfl_sync(0xffffffffu, at, 0);
                    if (at < BIG_CAP) continue;   // queued for the CTA-wide pass
                }
                const int32_t pz = A.pos[z];
                for (int64_t e = e0 + lane; e < e1; e += 32) edge(e, pz);
            }
            __syncthreads();
            const int nbig = min(s_nbig, BIG_CAP);
            for (int bi = 0; bi < nbig; bi++) {
                const int32_t z = s_big[bi];
                const int32_t pz = A.pos[z];
                const int64_t e0 = A.ioff[z], e1 = e0 + A.icnt[z];
                for (int64_t e = e0 + tid; e < e1; e += GB) edge(e, pz);
            }
        }
        __syncthreads();
        // top-down over b's ancestors: x_w(y) -= sum of deposits above y.  A pair cut has no
        // chain (b's parent is the root and the root keeps no deposit reader above it).
        if (!pair && s_nch <= CHAIN_CAP) {
            // warp 0, 32 chain positions per step from the root down: the deposits are loaded
            // together and every lane re-adds them in chain order (the serial sum, bit for bit)
            if (tid < 32) {
                const int nch = s_nch;
                double run = 0.0;
                for (int top = nch - 1; top >= 0; top -= 32) {
                    const int c = top - tid;
                    const int32_t y = c >= 0 ? s_chain[c] : -1;
                    const double dep = y >= 0 ? A.accl[y] : 0.0;
                    double before = 0.0;
#pragma unroll 8
                    for (int j = 0; j < 32; j++) {
                        const double dj = __shfl_sync(0xffffffffu, dep, j);
                        if (j == tid) before = run;
                        if (top - j >= 0) run += dj;
                    }
                    if (y >= 0) {
                        if (before != 0.0) {
                            A.xw[y] -= before;
                            mark_dirty(y, gflag, dirty, &s_ndirty, &s_overflow);
                        }
                        A.accl[y] = 0.0;
                    }
                }
            }
        } else if (tid == 0) {
            if (pair) {
                // pair cut: the chain is the root alone
                const int32_t y = r;
                A.accl[y] = 0.0;
            } else {   // very deep chain: per-node suffix via repeated upward walks
                for (int32_t y = xpar;; y = A.a[y]) {
                    double above = 0.0;
                    for (int32_t z2 = A.a[y]; z2 != y; z2 = A.a[z2]) {
                        above += A.accl[z2];
                        if (z2 == r) break;
                    }
                    if (y != r && above != 0.0) {
                        A.xw[y] -= above;
                        mark_dirty(y, gflag, dirty, &s_ndirty, &s_overflow);
                    }
                    if (y == r) break;
                }
                for (int32_t y = xpar;; y = A.a[y]) {
                    A.accl[y] = 0.0;
                    if (y == r) break;
                }
            }
        }
        __syncthreads();
        sec(4);
        // ---- record the split and its child part
        if (bsize <= O.small_part) {
            // ordered compaction of b's members (DFS order) + in-part subtree sizes
            __shared__ int s_off;
            if (tid == 0) s_off = atomicAdd(O.alloc, bsize);
            __syncthreads();
            const int off = s_off;
            int base = 0;
            for (int64_t k0 = blo; k0 < bhi; k0 += GB) {
                const int64_t k = k0 + tid;
                const int32_t x = k < bhi ? A.order[k] : 0;
                const int f = (k < bhi && A.gmark[x] == pid_b) ? 1 : 0;
                // block exclusive scan of f
                int inc = f;
                const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += v;
                }
                if (lane == 31) si[wid] = inc;
                __syncthreads();
                if (wid == 0) {
                    int v = si[lane];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int w2 = __shfl_up_sync(0xffffffffu, v, o);
                        if (lane >= o) v += w2;
                    }
                    si[lane] = v;   // inclusive warp totals
                }
                __syncthreads();
                const int before = (wid ? si[wid - 1] : 0) + inc - f;
                if (f) {
                    O.pbuf2[off + base + before] = x;
                    O.posb[off + base + before] = A.pos[x];
                }
                base += si[GB / 32 - 1];
                __syncthreads();
            }
            for (int t = tid; t < bsize; t += GB) {
                const int32_t y = O.pbuf2[off + t];
                const int32_t endp = O.posb[off + t] + A.sz[y];
                int lo2 = t, hi2 = bsize;
                while (lo2 < hi2) {
                    const int mid = (lo2 + hi2) >> 1;
                    if (O.posb[off + mid] < endp) lo2 = mid + 1;
                    else hi2 = mid;
                }
                O.psz[y] = lo2 - t;
            }
            if (tid == 0) {
                const int di = atomicAdd(O.ndesc, 1);
                PartDesc d;
                d.off = off;
                d.len = bsize;
                d.from_layout = 0;
                d.pad = 0;
                O.desc[di] = d;
                const int li = atomicAdd(O.nlog, 1);
                O.log_pid[li] = pid;
                O.log_seq[li] = seq;
                O.log_gain[li] = gain;
                O.log_kind[li] = 0;
                O.log_child[li] = di;
            }
        } else if (tid == 0) {
            const int ni = atomicAdd(O.nnext, 1);
            O.nx_lo[ni] = blo;
            O.nx_hi[ni] = bhi;
            O.nx_pid[ni] = pid_b;
            O.nx_root[ni] = xc;
            O.nx_size[ni] = bsize;
            const int li = atomicAdd(O.nlog, 1);
            O.log_pid[li] = pid;
            O.log_seq[li] = seq;
            O.log_gain[li] = gain;
            O.log_kind[li] = 1;
            O.log_child[li] = pid_b;
        }
        seq++;
        __syncthreads();
        sec(5);
    }
    // leave the flag arrays clean for the next part on this SM
    __syncthreads();
    if (tid == 0) {
        atomicMax(O.unresolved + 3, (unsigned long long)seq);
        atomicMax(O.unresolved + 4, (unsigned long long)(clock64() - t_cta));
    }
    for (int t = tid; t < min(s_ndirty, DIRTY_CAP); t += GB) gflag[dirty[t]] = 0;
    for (int t = tid; t < s_ntop; t += GB) gflag[tx[t]] = 0;
    for (int t = tid; t < s_nneg; t += GB) negflag[negl[t]] = 0;
}

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
    k_positive<<<grid_for(np * 32, 128, SMS() * 64), 128, 0, s>>>(A);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(hng.data(), ngains.p, np * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(hun.data(), nunres.p, np * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
}

struct PosScratch {
    DBuf<int32_t> pbuf, pbuf2, tbuf, pmark, ppos, psz, gmark, flags;
    DBuf<int2> sstk, sstk2;
    DBuf<double> wpart, dep, pso, psi, pdp, gbuf, gbuf2, xw, sob, sib;
    DBuf<int32_t> neg_pool, log_pid, log_seq, log_kind, log_child, cnt6, nx_pid, nx_root, nx_size,
        posb, nch;
    DBuf<double> log_gain, vso, vsi, vdp, pso2, psi2, pdp2;
    DBuf<int64_t> nx_lo, nx_hi, choff, chunks;
    DBuf<PartDesc> desc;
    DBuf<uint8_t> gflag, negflag;
    DBuf<unsigned long long> unres_d;
    DBuf<GSlice> slices;
    DBuf<int32_t> dirty_pool;
    DBuf<GPart> dparts2;
    DBuf<double> accl;
    DBuf<int64_t> ioff, icnt_flat, ioff_flat;
    DBuf<int32_t> icnt, iz, iy;
    DBuf<double> iu;
};

void run_positive(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m, int64_t scc_cap,
                  int64_t *splits, int64_t *unresolved, int *changed, std::vector<double> *gains) {
    cudaStream_t s = ctx->stream;
    const int64_t n = G.n, nc = F.n_comms;
    *splits = 0;
    *unresolved = 0;
    *changed = 0;
    if (gains) gains->clear();
    if (m == 0.0 || n == 0) return;
    const double t_call = now_ms();
    const bool plog = getenv("SLM_POS_LOG") != nullptr;
    double tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    auto tmark = [&](int k) {
        if (!plog) return;
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        tp[k] = now_ms();
    };
    read_small_part();
    phase_mark(ctx, -1);
    CTX_SCRATCH(DBuf<uint8_t>, bad);   // grow-only scratch kept across calls
    bad.resize(nc);
    CUDA_TRY(cudaMemsetAsync(bad.p, 0, nc, s));
    static const bool no_wown = getenv("SLM_WOWN") && atoi(getenv("SLM_WOWN")) == 0;
    if (!no_wown && ctx->wown_version == F.version && G.u32_ok && ctx->wown.n == (size_t)n) {
        wown_to_node_order(ctx, G);
        run_local_gains_wown(ctx, G, F, m, ctx->wown.p, nullptr, bad.p);
    }
    else
        run_local_gains(ctx, G, F, m, nullptr, bad.p);
    CTX_SCRATCH(DBuf<int32_t>, f);
    CTX_SCRATCH(DBuf<int32_t>, pos);
    CTX_SCRATCH(DBuf<int32_t>, list);
    f.resize(nc + 1);
    pos.resize(nc + 1);
    CUDA_TRY(cudaMemsetAsync(f.p + nc, 0, 4, s));
    k_bad_flags<<<grid_for(nc, 256), 256, 0, s>>>(bad.p, nc, f.p);
    dev_exclusive_sum<int32_t, int32_t>(ctx, f.p, pos.p, nc + 1);
    int32_t nbad = 0;
    CUDA_TRY(cudaMemcpyAsync(&nbad, pos.p + nc, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (nbad == 0) return;
    list.resize(nbad);
    k_bad_scatter<<<grid_for(nc, 256), 256, 0, s>>>(f.p, pos.p, nc, list.p);
    phase_mark(ctx, PH_POS_LG);
    tmark(0);
    // bad community ids and their layout ranges (only those: cptr itself stays on the device)
    std::vector<int32_t> hbad(nbad);
    std::vector<int2> hrng(nbad);
    std::vector<uint8_t> hheavy(nbad, 0);
    {
        CTX_SCRATCH(DBuf<int2>, drng);
        drng.resize(nbad);
        k_bad_ranges<<<grid_for(nbad, 256), 256, 0, s>>>(list.p, nbad, F.cptr.p, drng.p);
        CUDA_TRY(cudaMemcpyAsync(hrng.data(), drng.p, nbad * 8, cudaMemcpyDeviceToHost, s));
        // heavy nodes of this level (found once per level graph)
        if (!G.heavy_valid) {
            DBuf<int32_t> hf, hp;
            hf.resize(n + 1);
            hp.resize(n + 1);
            CUDA_TRY(cudaMemsetAsync(hf.p + n, 0, 4, s));
            k_heavy_flags<<<grid_for(n, 256), 256, 0, s>>>(G.uptr.p, n, HEAVY_DEG, hf.p);
            dev_exclusive_sum<int32_t, int32_t>(ctx, hf.p, hp.p, n + 1);
            int32_t nh = 0;
            CUDA_TRY(cudaMemcpyAsync(&nh, hp.p + n, 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            G.heavy_nodes.resize(nh > 0 ? nh : 1);
            if (nh) k_heavy_scatter<<<grid_for(n, 256), 256, 0, s>>>(hf.p, hp.p, n, G.heavy_nodes.p);
            G.heavy_n = nh;
            G.heavy_valid = true;
            CUDA_TRY(cudaStreamSynchronize(s));
        }
        if (G.heavy_n) {
            CTX_SCRATCH(DBuf<uint8_t>, hc);
            CTX_SCRATCH(DBuf<uint8_t>, hb);
            hc.resize(nc);
            hb.resize(nbad);
            CUDA_TRY(cudaMemsetAsync(hc.p, 0, nc, s));
            k_heavy_mark<<<grid_for(G.heavy_n, 256), 256, 0, s>>>(G.heavy_nodes.p, G.heavy_n,
                                                                  F.comm.p, hc.p);
            k_bad_heavy<<<grid_for(nbad, 256), 256, 0, s>>>(list.p, nbad, hc.p, hb.p);
            CUDA_TRY(cudaMemcpyAsync(hheavy.data(), hb.p, nbad, cudaMemcpyDeviceToHost, s));
        }
    }
    CUDA_TRY(cudaMemcpyAsync(hbad.data(), list.p, nbad * 4, cudaMemcpyDeviceToHost, s));
    CTX_SCRATCH(DBuf<uint32_t>, g_stamp);   // monotone part stamps (never reset)
    if (g_stamp.p == nullptr) {
        g_stamp.resize(1);
        CUDA_TRY(cudaMemsetAsync(g_stamp.p, 0, 4, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    // n-sized scratch, kept across calls (grow-only; pmark holds monotone stamps, so it is
    // cleared only when reallocated)
    CTX_SCRATCH(PosScratch, SC);
    DBuf<int32_t> &pbuf = SC.pbuf, &pbuf2 = SC.pbuf2, &tbuf = SC.tbuf, &pmark = SC.pmark,
                  &ppos = SC.ppos, &psz = SC.psz, &gmark = SC.gmark, &flags = SC.flags;
    DBuf<int2> &sstk = SC.sstk, &sstk2 = SC.sstk2;
    DBuf<double> &wpart = SC.wpart, &dep = SC.dep, &pso = SC.pso, &psi = SC.psi, &pdp = SC.pdp,
                 &gbuf = SC.gbuf, &gbuf2 = SC.gbuf2, &xw = SC.xw, &sob = SC.sob, &sib = SC.sib;
    const bool fresh_pmark = pmark.cap < (size_t)n;
    pbuf.resize(n); pbuf2.resize(n); tbuf.resize(n); pmark.resize(n); ppos.resize(n);
    psz.resize(n); gmark.resize(n); sstk.resize(n); sstk2.resize(n);
    wpart.resize(n); dep.resize(n); pso.resize(n); psi.resize(n); pdp.resize(n);
    gbuf.resize(n); gbuf2.resize(n);
    flags.resize(2);
    if (fresh_pmark) CUDA_TRY(cudaMemsetAsync(pmark.p, 0, n * 4, s));
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
    tmark(1);
    // 1. small bad communities straight from the layout
    std::vector<PartDesc> small1;
    std::vector<int64_t> order_kind(nbad);   // >=0: small1 index, <0: -(giant id)-1
    std::vector<int64_t> giant_of;
    std::vector<int32_t> giant_comm;   // bad-list indices of the giant communities
    // a part goes to the warp executor when it is small and holds no heavy member (a warp
    // rescans every member row at each split: coarse levels have hub members whose rows hold
    // millions of entries, which the CTA executor processes cooperatively)
    // communities whose assignment cycle is longer than 2 (never produced by run(), F5)
    // take the literal executor (slm_positive_lit.cu); the fast executors assume <= 2
    std::vector<int32_t> clen;
    bad_cycle_lengths(ctx, F, list.p, nbad, clen);
    std::vector<int2> lit_rng;
    constexpr int64_t LIT_BASE = -(int64_t(1) << 40);
    for (int32_t i = 0; i < nbad; i++) {
        int32_t sz = hrng[i].y - hrng[i].x;
        if (clen[i] > 2) {
            order_kind[i] = LIT_BASE - (int64_t)lit_rng.size();
            lit_rng.push_back(hrng[i]);
            continue;
        }
        if (sz <= SMALL_PART && !hheavy[i]) {
            PartDesc d;
            d.off = hrng[i].x;
            d.len = sz;
            d.from_layout = 1;
            d.pad = 0;
            order_kind[i] = (int64_t)small1.size();
            small1.push_back(d);
        } else {
            order_kind[i] = -1 - (int64_t)giant_comm.size();
            giant_comm.push_back(i);   // index into hbad / hrng
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
    // 2. giant communities: one CTA per part with incremental state (k_giant_cta), in waves
    //    (a cut subtree larger than SMALL_PART becomes a part of the next wave); small cut
    //    subtrees are collected for a second warp-executor batch
    tmark(2);
    std::vector<PartDesc> small2;
    std::vector<int32_t> l_pid, l_seq, l_kind, l_child;
    std::vector<double> l_gain;
    std::vector<int32_t> giant_pid;   // per giant community (in bad-list order)
    bool gchanged = false;
    int64_t gunres = 0;
    if (!giant_comm.empty()) {
        xw.resize(n);
        sob.resize(n);
        sib.resize(n);
        GiantArgs GA;
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
        if (SC.accl.cap < (size_t)n) {
            SC.accl.resize(n);
            CUDA_TRY(cudaMemsetAsync(SC.accl.p, 0, n * 8, s));
        }
        SC.accl.resize(n);
        GA.accl = SC.accl.p;
        SC.ioff.resize(n);
        SC.icnt.resize(n);
        GA.ioff = SC.ioff.p;
        GA.icnt = SC.icnt.p;
        GA.iz = nullptr;
        GA.iu = nullptr;
        GA.iy = nullptr;
        int64_t nintra_w0 = 0;
        bool first_wave = true;
        GA.m = m;
        GA.m2 = m * m;
        k_init_i32<<<grid_for(n, 256), 256, 0, s>>>(gmark.p, n, 0);
        // pools
        DBuf<int32_t> &neg_pool = SC.neg_pool, &log_pid = SC.log_pid, &log_seq = SC.log_seq,
                      &log_kind = SC.log_kind, &log_child = SC.log_child, &cnt6 = SC.cnt6,
                      &nx_pid = SC.nx_pid, &nx_root = SC.nx_root, &nx_size = SC.nx_size,
                      &posb = SC.posb;
        DBuf<double> &log_gain = SC.log_gain, &vso = SC.vso, &vsi = SC.vsi, &vdp = SC.vdp,
                     &pso2 = SC.pso2, &psi2 = SC.psi2, &pdp2 = SC.pdp2;
        DBuf<int64_t> &nx_lo = SC.nx_lo, &nx_hi = SC.nx_hi;
        DBuf<PartDesc> &desc = SC.desc;
        DBuf<uint8_t> &gflag = SC.gflag, &negflag = SC.negflag;
        DBuf<unsigned long long> &unres_d = SC.unres_d;
        neg_pool.resize(n);
        log_pid.resize(n);
        log_seq.resize(n);
        log_kind.resize(n);
        log_child.resize(n);
        log_gain.resize(n);
        desc.resize(n);
        nx_lo.resize(n);
        nx_hi.resize(n);
        nx_pid.resize(n);
        nx_root.resize(n);
        nx_size.resize(n);
        posb.resize(n);
        gflag.resize(n + 4);
        negflag.resize(n + 4);
        cnt6.resize(6);   // nlog, ndesc, alloc, nnext, pid_ctr, pad
        unres_d.resize(8);
        CUDA_TRY(cudaMemsetAsync(gflag.p, 0, n + 4, s));
        CUDA_TRY(cudaMemsetAsync(negflag.p, 0, n + 4, s));
        CUDA_TRY(cudaMemsetAsync(cnt6.p, 0, 24, s));
        CUDA_TRY(cudaMemsetAsync(unres_d.p, 0, 64, s));
        GOut O;
        O.log_pid = log_pid.p;
        O.log_seq = log_seq.p;
        O.log_kind = log_kind.p;
        O.log_child = log_child.p;
        O.log_gain = log_gain.p;
        O.nlog = cnt6.p + 0;
        O.desc = desc.p;
        O.ndesc = cnt6.p + 1;
        O.pbuf2 = pbuf2.p;
        O.posb = posb.p;
        O.psz = psz.p;
        O.alloc = cnt6.p + 2;
        O.nx_lo = nx_lo.p;
        O.nx_hi = nx_hi.p;
        O.nx_pid = nx_pid.p;
        O.nx_root = nx_root.p;
        O.nx_size = nx_size.p;
        O.nnext = cnt6.p + 3;
        O.pid_ctr = cnt6.p + 4;
        O.unresolved = unres_d.p;
        O.flags = flags.p;
        O.small_part = SMALL_PART;
        CTX_SCRATCH(DBuf<unsigned long long>, gprof);
        O.prof = nullptr;
        if (plog) {
            gprof.resize(8 + 8 * 4096);
            CUDA_TRY(cudaMemsetAsync(gprof.p, 0, gprof.bytes(), s));
            O.prof = gprof.p;
        }
        // wave 0: the giant bad communities
        std::vector<GPart> wave;
        int32_t next_pid = 1;
        int64_t neg_alloc = 0;
        for (int32_t c : giant_comm) {
            GPart gp;
            gp.lo = hrng[c].x;
            gp.hi = hrng[c].y;
            gp.cbase = hrng[c].x;
            gp.pid = next_pid++;
            gp.neg_off = neg_alloc;
            neg_alloc += gp.hi - gp.lo;
            giant_pid.push_back(gp.pid);
            k_g_mark<<<grid_for(gp.hi - gp.lo, 256), 256, 0, s>>>(F.order.p, gp.lo, gp.hi, gp.pid,
                                                                   gmark.p);
            wave.push_back(gp);
        }
        {   // roots: the first layout member of each community
            std::vector<int32_t> roots(wave.size());
            for (size_t i = 0; i < wave.size(); i++)
                CUDA_TRY(cudaMemcpyAsync(&roots[i], F.order.p + wave[i].lo, 4,
                                         cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            for (size_t i = 0; i < wave.size(); i++) wave[i].root = roots[i];
        }
        CUDA_TRY(cudaMemcpyAsync(cnt6.p + 4, &next_pid, 4, cudaMemcpyHostToDevice, s));
        DBuf<GPart> &dparts2 = SC.dparts2;
        DBuf<int32_t> &dirty_pool = SC.dirty_pool;
        tmark(6);
        while (!wave.empty()) {
            tmark(6);
            // init pass of every part of the wave, batched: w_part, LCA deposits, subtree
            // sums (one exclusive scan over the concatenated slices), part totals
            const int ns = (int)wave.size();
            std::vector<GSlice> hs(ns);
            int64_t N = 0;
            for (int i = 0; i < ns; i++) {
                hs[i].lo = wave[i].lo;
                hs[i].hi = wave[i].hi;
                hs[i].cbase = wave[i].cbase;
                hs[i].flat = N;
                hs[i].pid = wave[i].pid;
                hs[i].pad = 0;
                N += wave[i].hi - wave[i].lo;
            }
            SC.slices.resize(ns);
            CUDA_TRY(cudaMemcpyAsync(SC.slices.p, hs.data(), ns * sizeof(GSlice),
                                     cudaMemcpyHostToDevice, s));
            const GSlice *dsl = SC.slices.p;
            SC.nch.resize(N + 1);
            SC.choff.resize(N + 1);
            CUDA_TRY(cudaMemsetAsync(SC.nch.p + N, 0, 4, s));
            const int build_intra = first_wave ? 1 : 0;
            k_gb_chunks<<<grid_for(N, 256), 256, 0, s>>>(GA, dsl, ns, N, SC.nch.p, build_intra);
            dev_exclusive_sum<int32_t, int64_t>(ctx, SC.nch.p, SC.choff.p, N + 1);
            int64_t nck = 0;
            CUDA_TRY(cudaMemcpyAsync(&nck, SC.choff.p + N, 8, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            SC.chunks.resize(std::max<int64_t>(1, nck));
            k_gb_expand<<<grid_for(N, 256), 256, 0, s>>>(GA, dsl, ns, N, SC.nch.p, SC.choff.p,
                                                        SC.chunks.p);
            const unsigned GW = grid_for(nck * 32, 256, SMS() * 32);
            k_gb_wpart<<<GW, 256, 0, s>>>(GA, dsl, ns, SC.chunks.p, nck, build_intra);
            if (build_intra) {   // intra-part adjacency lists of the wave-0 members
                SC.icnt_flat.resize(N + 1);
                SC.ioff_flat.resize(N + 1);
                k_gb_icount<<<grid_for(N, 256), 256, 0, s>>>(GA, dsl, ns, N, SC.icnt_flat.p);
                CUDA_TRY(cudaMemsetAsync(SC.icnt_flat.p + N, 0, 8, s));
                dev_exclusive_sum<int64_t, int64_t>(ctx, SC.icnt_flat.p, SC.ioff_flat.p, N + 1);
                int64_t nintra = 0;
                CUDA_TRY(cudaMemcpyAsync(&nintra, SC.ioff_flat.p + N, 8, cudaMemcpyDeviceToHost, s));
                CUDA_TRY(cudaStreamSynchronize(s));
                SC.iz.resize(std::max<int64_t>(1, nintra));
                SC.iu.resize(std::max<int64_t>(1, nintra));
                GA.iz = SC.iz.p;
                GA.iu = SC.iu.p;
                // entry owners for the flat LCA pass; lists beyond 2^27 entries (a giant part
                // spanning most of the graph) keep the warp-per-row pass and its memory
                nintra_w0 = nintra <= (int64_t(1) << 27) ? nintra : 0;
                if (nintra_w0 > 0) {
                    SC.iy.resize(nintra_w0);
                    GA.iy = SC.iy.p;
                } else {
                    SC.iy.release();
                    GA.iy = nullptr;
                }
                k_gb_ioff<<<grid_for(N, 256), 256, 0, s>>>(GA, dsl, ns, N, SC.ioff_flat.p);
                k_gb_ifill<<<GW, 256, 0, s>>>(GA, dsl, ns, SC.chunks.p, nck);
                first_wave = false;
            }
            k_gb_dep<<<grid_for(N, 256), 256, 0, s>>>(GA, dsl, ns, N);
            if (build_intra && nintra_w0 > 0 && getenv("SLM_LCA_CHUNKS") == nullptr)
                k_gb_lca_flat<<<grid_for(nintra_w0, 256, SMS() * 32), 256, 0, s>>>(GA, nintra_w0);
            else
                k_gb_lca<<<GW, 256, 0, s>>>(GA, dsl, ns, SC.chunks.p, nck);
            vso.resize(N + 1);
            vsi.resize(N + 1);
            vdp.resize(N + 1);
            pso2.resize(N + 1);
            psi2.resize(N + 1);
            pdp2.resize(N + 1);
            k_gb_gather<<<grid_for(N, 256), 256, 0, s>>>(GA, dsl, ns, N, vso.p, vsi.p, vdp.p);
            CUDA_TRY(cudaMemsetAsync(vso.p + N, 0, 8, s));
            CUDA_TRY(cudaMemsetAsync(vsi.p + N, 0, 8, s));
            CUDA_TRY(cudaMemsetAsync(vdp.p + N, 0, 8, s));
            dev_exclusive_sum<double, double>(ctx, vso.p, pso2.p, N + 1);
            dev_exclusive_sum<double, double>(ctx, vsi.p, psi2.p, N + 1);
            dev_exclusive_sum<double, double>(ctx, vdp.p, pdp2.p, N + 1);
            k_gb_subsums<<<grid_for(N, 256), 256, 0, s>>>(GA, dsl, ns, N, pso2.p, psi2.p, pdp2.p);
            tmark(7);
            tp[3] += tp[7] - tp[6];
            const int64_t np = (int64_t)wave.size();
            dirty_pool.resize(np * DIRTY_CAP);
            for (int64_t i = 0; i < np; i++) wave[i].dirty_off = i * DIRTY_CAP;
            dparts2.resize(np);
            CUDA_TRY(cudaMemcpyAsync(dparts2.p, wave.data(), np * sizeof(GPart),
                                     cudaMemcpyHostToDevice, s));
            k_gb_totals<<<(unsigned)((np + 127) / 128), 128, 0, s>>>(dsl, ns, pso2.p, psi2.p,
                                                                     dparts2.p);
            CUDA_TRY(cudaMemsetAsync(cnt6.p + 3, 0, 4, s));
            if (!ctx->giant_attr_set) {
                CUDA_TRY(cudaFuncSetAttribute(k_giant_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)GSMEM));
                ctx->giant_attr_set = true;
            }
            k_giant_cta<<<(unsigned)np, GB, GSMEM, s>>>(GA, dparts2.p, O, neg_pool.p, dirty_pool.p,
                                                    gflag.p, negflag.p);
            CUDA_TRY(cudaGetLastError());
            int32_t nnext = 0;
            CUDA_TRY(cudaMemcpyAsync(&nnext, cnt6.p + 3, 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            if (plog) tp[4] += now_ms() - tp[7];
            wave.clear();
            if (nnext > 0) {
                std::vector<int64_t> hlo(nnext), hhi(nnext);
                std::vector<int32_t> hpid(nnext), hroot(nnext), hsize(nnext);
                CUDA_TRY(cudaMemcpyAsync(hlo.data(), nx_lo.p, nnext * 8, cudaMemcpyDeviceToHost, s));
                CUDA_TRY(cudaMemcpyAsync(hhi.data(), nx_hi.p, nnext * 8, cudaMemcpyDeviceToHost, s));
                CUDA_TRY(cudaMemcpyAsync(hpid.data(), nx_pid.p, nnext * 4, cudaMemcpyDeviceToHost, s));
                CUDA_TRY(cudaMemcpyAsync(hroot.data(), nx_root.p, nnext * 4, cudaMemcpyDeviceToHost, s));
                CUDA_TRY(cudaMemcpyAsync(hsize.data(), nx_size.p, nnext * 4, cudaMemcpyDeviceToHost, s));
                CUDA_TRY(cudaStreamSynchronize(s));
                neg_alloc = 0;
                for (int32_t i = 0; i < nnext; i++) {
                    GPart gp;
                    gp.lo = hlo[i];
                    gp.hi = hhi[i];
                    gp.cbase = hlo[i] - 0;   // slice start in community coordinates below
                    gp.pid = hpid[i];
                    gp.root = hroot[i];
                    gp.neg_off = neg_alloc;
                    neg_alloc += hsize[i];
                    wave.push_back(gp);
                }
                // cbase: the community layout base of the part (pos[] is community-relative)
                std::vector<int32_t> prs(wave.size());
                for (size_t i = 0; i < wave.size(); i++)
                    CUDA_TRY(cudaMemcpyAsync(&prs[i], F.pos.p + wave[i].root, 4,
                                             cudaMemcpyDeviceToHost, s));
                CUDA_TRY(cudaStreamSynchronize(s));
                for (size_t i = 0; i < wave.size(); i++) wave[i].cbase = wave[i].lo - prs[i];
            }
        }
        int32_t hc[4];
        unsigned long long hun = 0, hst[8];
        if (plog) {
            CUDA_TRY(cudaMemcpyAsync(hst, unres_d.p, 64, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            fprintf(stderr, "[giant] full passes %llu scanned %llu max splits/part %llu max cycles "
                    "%llu\n", hst[1], hst[2], hst[3], hst[4]);
            unsigned long long hp[8];
            CUDA_TRY(cudaMemcpy(hp, O.prof, 64, cudaMemcpyDeviceToHost));
            fprintf(stderr, "[giant] section cycles: incr %llu full %llu neg %llu cut %llu edges %llu "
                    "record %llu | rest-edges %llu walk steps %llu\n", hp[0], hp[1], hp[2],
                    hp[3], hp[4], hp[5], hp[6], hp[7]);
            std::vector<unsigned long long> pc(8 * 4096);
            CUDA_TRY(cudaMemcpy(pc.data(), O.prof + 8, pc.size() * 8, cudaMemcpyDeviceToHost));
            int wb = 0;
            unsigned long long wt = 0;
            for (int b = 0; b < 4096; b++) {
                unsigned long long t = 0;
                for (int k = 0; k < 6; k++) t += pc[8 * b + k];
                if (t > wt) { wt = t; wb = b; }
            }
            fprintf(stderr, "[giant] slowest CTA %d: incr %llu full %llu neg %llu cut %llu edges %llu "
                    "record %llu\n", wb, pc[8 * wb], pc[8 * wb + 1], pc[8 * wb + 2], pc[8 * wb + 3],
                    pc[8 * wb + 4], pc[8 * wb + 5]);
        }
        CUDA_TRY(cudaMemcpyAsync(hc, cnt6.p, 16, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(&hun, unres_d.p, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        const int32_t nlog = hc[0], ndesc = hc[1];
        gunres = (int64_t)hun;
        gchanged = nlog > 0;
        small2.resize(ndesc);
        if (ndesc)
            CUDA_TRY(cudaMemcpyAsync(small2.data(), desc.p, ndesc * sizeof(PartDesc),
                                     cudaMemcpyDeviceToHost, s));
        l_pid.resize(nlog);
        l_seq.resize(nlog);
        l_kind.resize(nlog);
        l_child.resize(nlog);
        l_gain.resize(nlog);
        if (nlog) {
            CUDA_TRY(cudaMemcpyAsync(l_pid.data(), log_pid.p, nlog * 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(l_seq.data(), log_seq.p, nlog * 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(l_kind.data(), log_kind.p, nlog * 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(l_child.data(), log_child.p, nlog * 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(l_gain.data(), log_gain.p, nlog * 8, cudaMemcpyDeviceToHost, s));
        }
        CUDA_TRY(cudaStreamSynchronize(s));
        tot += nlog;
        un += gunres;
        // small parts cut from giants (their own regions in pbuf2 / sstk2 / gbuf2)
        A.pbuf = pbuf2.p;
        A.sstk = sstk2.p;
        A.gains = gbuf2.p;
        launch_small(ctx, A, small2, dparts, ngains, nunres, hng2, hun2);
        for (size_t i = 0; i < small2.size(); i++) {
            tot += hng2[i];
            un += hun2[i];
        }
    }
    int32_t hflags[2];
    CUDA_TRY(cudaMemcpyAsync(hflags, flags.p, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (getenv("SLM_POS_LOG")) {
        int64_t gm = 0;
        for (int32_t c : giant_comm) gm += hrng[c].y - hrng[c].x;
        fprintf(stderr, "[positive] bad %d (small %zu) giant %zu members %lld | giant splits %zu "
                "unresolved %lld small2 %zu | total splits %lld unres %lld | %.1f ms: lg %.1f "
                "alloc %.1f small1 %.1f ginit %.1f gcta %.1f\n", nbad,
                small1.size(), giant_comm.size(), (long long)gm, l_pid.size(), (long long)gunres,
                small2.size(), (long long)tot, (long long)un, now_ms() - t_call, tp[0] - t_call,
                tp[1] - tp[0], tp[2] - tp[1], tp[3], tp[4]);
    }
    phase_mark(ctx, PH_POS_GIANT);
    SLM_REQUIRE(!hflags[1], SLM_EUNSUP, "assignment cycle longer than 2 in POSITIVE");
    std::vector<std::vector<double>> lit_gains;
    std::vector<int32_t> lit_unres, lit_changed;
    int64_t lit_warn = 0;
    run_positive_literal(ctx, G, F, m, scc_cap, lit_rng, lit_gains, lit_unres, lit_changed,
                         &lit_warn);
    bool lchanged = false;
    for (size_t j = 0; j < lit_rng.size(); j++) {
        tot += (int64_t)lit_gains[j].size();
        un += lit_unres[j];
        lchanged |= lit_changed[j] != 0;
    }
    ctx->last_pos_warnings = lit_warn;
    *splits = tot;
    *unresolved = un;
    *changed = hflags[0] || gchanged || lchanged;
    if (gains && tot > 0) {
        // the reference's order: communities ascending; within a community its LIFO stack,
        // i.e. a cut's gain, then the cut subtree's gains, then the rest's
        std::vector<double> hg1(n), hg2(n);
        CUDA_TRY(cudaMemcpyAsync(hg1.data(), gbuf.p, n * 8, cudaMemcpyDeviceToHost, s));
        if (!small2.empty())
            CUDA_TRY(cudaMemcpyAsync(hg2.data(), gbuf2.p, n * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        // split logs per giant part, in sequence order
        std::map<int32_t, std::vector<std::pair<int32_t, size_t>>> by_pid;
        for (size_t li = 0; li < l_pid.size(); li++) by_pid[l_pid[li]].push_back({l_seq[li], li});
        for (auto &kv : by_pid) std::sort(kv.second.begin(), kv.second.end());
        std::function<void(int32_t)> emit = [&](int32_t pid) {
            auto it = by_pid.find(pid);
            if (it == by_pid.end()) return;
            for (auto &sl : it->second) {
                const size_t li = sl.second;
                gains->push_back(l_gain[li]);
                if (l_kind[li] == 0) {
                    const PartDesc &d = small2[l_child[li]];
                    for (int k = 0; k < hng2[l_child[li]]; k++) gains->push_back(hg2[d.off + k]);
                } else {
                    emit(l_child[li]);
                }
            }
        };
        for (int32_t i = 0; i < nbad; i++) {
            if (order_kind[i] <= LIT_BASE) {
                const auto &lg = lit_gains[LIT_BASE - order_kind[i]];
                gains->insert(gains->end(), lg.begin(), lg.end());
            } else if (order_kind[i] >= 0) {
                const PartDesc &d = small1[order_kind[i]];
                for (int k = 0; k < hng1[order_kind[i]]; k++) gains->push_back(hg1[d.off + k]);
            } else {
                emit(giant_pid[-1 - order_kind[i]]);
            }
        }
    }
}

// a kernel of this translation unit (module preloading, slm_capi.cu preload_modules)
const void *slm_anchor_positive() { return (const void *)k_positive; }
