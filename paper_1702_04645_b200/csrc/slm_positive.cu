// slm_positive.cu -- POSITIVE correction (positive_correction, detector.py:338-362;
// _split_community 197-285; _detach_gain 178-194; _best_pair_cut 288-335).
//
// One warp per bad community (a community with a member of negative local gain), walking
// the reference's LIFO stack of parts.  Parts are kept as contiguous slices of the
// community's DFS pre-order (slm_forest.cu): a branch subtree is a sub-slice, and cutting it
// out leaves the rest in DFS order with the cut subtree's size subtracted along its
// ancestor chain.  Per part, every branch-cut gain comes from one pass:
//   x_w(sub(x)) = sum_{v in sub(x)} dep[v],  dep[v] = w_part(v) - sum_{entries (y,z) with
//   LCA(y,z) = v} u  (prefix sums over the DFS slice),
// the null term from prefix sums of s_out / s_in, and the gain with the reference's exact
// fp64 operand order.  The chosen cut is the first strict maximum > 0 in ascending node id;
// a 2-cycle pair cut (cycles are <= 2) equals detaching the DFS subtree of the
// cycle's second node with both cycle nodes self-assigned.  Since parts are independent and
// each warp replays its community's stack exactly, the split sequence and the gains list
// order match the reference.
#include "slm_internal.cuh"
#include <cub/cub.cuh>

struct PosArgs {
    const int64_t *uptr;
    const int32_t *unbr;
    const double *uu;
    const double *s_out, *s_in;
    int32_t *a;
    const int32_t *cptr, *order, *sz0;
    const int32_t *bad;
    int64_t nbad;
    double m, m2;
    int32_t *pbuf, *tbuf, *pmark, *ppos, *psz;
    int2 *sstk;
    double *wpart, *dep, *pre_so, *pre_si, *pre_dep;
    double *gains;       // per community segment
    int32_t *ngains;     // per bad index
    int32_t *neg_unres;  // per bad index
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
__device__ double warp_exscan(const int32_t *P, int len, const double *val_of_node, double *out,
                              const double *node_vals_override) {
    const int lane = threadIdx.x & 31;
    double carry = 0.0;
    for (int cb = 0; cb < len; cb += 32) {
        int k = cb + lane;
        double v = 0.0;
        if (k < len) v = node_vals_override ? node_vals_override[P[k]] : val_of_node[P[k]];
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

__global__ void __launch_bounds__(128) k_positive(PosArgs A) {
    const int lane = threadIdx.x & 31;
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double m = A.m, m2 = A.m2;
    for (int64_t bi = w; bi < A.nbad; bi += nw) {
        const int32_t c = A.bad[bi];
        const int32_t base = A.cptr[c], size = A.cptr[c + 1] - base;
        for (int k = lane; k < size; k += 32) {
            int32_t x = A.order[base + k];
            A.pbuf[base + k] = x;
            A.psz[x] = A.sz0[x];
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
            // member gains against the part (detector.py:217-223)
            int neg = 0;
            for (int k = lane; k < len; k += 32) {
                int32_t x = P[k];
                double wp = 0.0;
                for (int64_t e = A.uptr[x]; e < A.uptr[x + 1]; e++)
                    if (A.pmark[A.unbr[e]] == (int32_t)stamp) wp += A.uu[e];
                A.wpart[x] = wp;
                A.dep[x] = wp;
                const double sox = A.s_out[x], six = A.s_in[x];
                double g = wp / m - (sox * (si_c - six) + six * (so_c - sox)) / m2;
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
            double tso = warp_exscan(P, len, A.s_out, pso, nullptr);
            double tsi = warp_exscan(P, len, A.s_in, psi, nullptr);
            double tdp = warp_exscan(P, len, A.dep, pdp, nullptr);
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

__global__ void k_bad_flags(const uint8_t *bad, int64_t nc, int32_t *f) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc;
         c += (int64_t)gridDim.x * blockDim.x)
        f[c] = bad[c] ? 1 : 0;
}
__global__ void k_bad_scatter(const int32_t *f, const int32_t *pos, int64_t nc, int32_t *list) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc;
         c += (int64_t)gridDim.x * blockDim.x)
        if (f[c]) list[pos[c]] = (int32_t)c;
}

static DBuf<uint32_t> g_stamp;   // monotone part stamps (never reset)

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
    if (g_stamp.p == nullptr) {
        g_stamp.resize(1);
        CUDA_TRY(cudaMemsetAsync(g_stamp.p, 0, 4, s));
    }
    DBuf<int32_t> pbuf, tbuf, pmark, ppos, psz, ngains, nunres, flags;
    DBuf<int2> sstk;
    DBuf<double> wpart, dep, pso, psi, pdp, gbuf;
    pbuf.resize(n);
    tbuf.resize(n);
    pmark.resize(n);
    ppos.resize(n);
    psz.resize(n);
    sstk.resize(n);
    wpart.resize(n);
    dep.resize(n);
    pso.resize(n);
    psi.resize(n);
    pdp.resize(n);
    gbuf.resize(n);
    ngains.resize(nbad);
    nunres.resize(nbad);
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
    A.cptr = F.cptr.p;
    A.order = F.order.p;
    A.sz0 = F.sz.p;
    A.bad = list.p;
    A.nbad = nbad;
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
    A.ngains = ngains.p;
    A.neg_unres = nunres.p;
    A.stamp_ctr = g_stamp.p;
    A.flags = flags.p;
    k_positive<<<grid_for((int64_t)nbad * 32, 128, 148LL * 64), 128, 0, s>>>(A);
    CUDA_TRY(cudaGetLastError());
    int32_t hflags[2];
    std::vector<int32_t> hng(nbad), hun(nbad), hbad(nbad), hcptr;
    CUDA_TRY(cudaMemcpyAsync(hflags, flags.p, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(hng.data(), ngains.p, nbad * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(hun.data(), nunres.p, nbad * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    SLM_REQUIRE(!hflags[1], SLM_EUNSUP, "assignment cycle longer than 2 in POSITIVE");
    int64_t tot = 0, un = 0;
    for (int64_t i = 0; i < nbad; i++) {
        tot += hng[i];
        un += hun[i];
    }
    *splits = tot;
    *unresolved = un;
    *changed = hflags[0];
    if (gains && tot > 0) {
        // gains in the reference's order: communities ascending, LIFO within each
        CUDA_TRY(cudaMemcpyAsync(hbad.data(), list.p, nbad * 4, cudaMemcpyDeviceToHost, s));
        hcptr.resize(nc + 1);
        CUDA_TRY(cudaMemcpyAsync(hcptr.data(), F.cptr.p, (nc + 1) * 4, cudaMemcpyDeviceToHost, s));
        std::vector<double> hg(n);
        CUDA_TRY(cudaMemcpyAsync(hg.data(), gbuf.p, n * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        for (int64_t i = 0; i < nbad; i++)
            for (int k = 0; k < hng[i]; k++) gains->push_back(hg[hcptr[hbad[i]] + k]);
    }
}
