// slm_positive_lit.cu -- POSITIVE for communities whose assignment cycle is longer than 2.
//
// run() never produces such cycles (ASSIGN's symmetric pairwise gain with the
// lowest-id tie-break rules them out, MAXIMAL only re-points into other trees, POSITIVE only
// self-assigns), so the fast executors of slm_positive.cu assume cycles <= 2.  A caller of
// positive_correction may pass any assignment forest, though, and the reference handles
// every cycle length (detector.py:197-335): branch cuts, the pair cut over arcs of the
// cycle, and -- for cycles longer than scc_cut_cap -- peeling the worst negative cycle node.
// This file restates that algorithm literally on the device, one community per CTA (lane 0
// runs it; these communities are rare and small), with the reference's summation orders:
// numpy pairwise sums over gathered operands (pw_sum_seq), Python left-to-right scalar
// expressions, no FMA.  Results (assignment, gains in LIFO order, unresolved counts) are
// therefore bit-identical to the reference for any weights.
#include "slm_internal.cuh"

namespace {

struct LitArgs {
    const int64_t *uptr;
    const int32_t *unbr;
    const double *uu;
    const double *s_out, *s_in;
    int32_t *a;
    double m, m2;
    int64_t scc_cap;
    int64_t *stamp;     // n: part stamp of each node (globally unique stamps)
    uint8_t *in_b;      // n
    int32_t *seen;      // n, -1 outside find_cycle
    int32_t *posof;     // n: index of a node inside its current part
    const int32_t *members;   // F.members (ascending ids per community)
};
struct LitJob {
    int64_t moff;       // members[moff .. moff + k)
    int32_t k;
    int64_t ip, dp;     // offsets into the int / double pools
    int64_t gp;         // gains offset
};
struct LitOut {
    int32_t ngains, unresolved, changed, nwarn;
};

__device__ void heapsort_i32(int32_t *v, int32_t n) {
    auto sift = [&](int32_t i, int32_t m) {
        for (;;) {
            int32_t c = 2 * i + 1;
            if (c >= m) return;
            if (c + 1 < m && v[c + 1] > v[c]) c++;
            if (v[i] >= v[c]) return;
            const int32_t t = v[i];
            v[i] = v[c];
            v[c] = t;
            i = c;
        }
    };
    for (int32_t i = n / 2 - 1; i >= 0; i--) sift(i, n);
    for (int32_t m = n - 1; m > 0; m--) {
        const int32_t t = v[0];
        v[0] = v[m];
        v[m] = t;
        sift(0, m);
    }
}

__device__ double gather_sum(const double *src, const int32_t *idx, int32_t k, double *tmp) {
    for (int32_t q = 0; q < k; q++) tmp[q] = src[idx[q]];
    return pw_sum_seq(tmp, k);
}

// children of the part's members restricted to the part (detector.py:229-233), by position
__device__ void part_children(const LitArgs &A, const int32_t *mem, int32_t pn, int64_t cur,
                              int32_t *chp, int32_t *chl, int32_t *fill) {
    for (int32_t q = 0; q <= pn; q++) chp[q] = 0;
    for (int32_t q = 0; q < pn; q++) {
        const int32_t x = mem[q], t = A.a[x];
        if (t != x && A.stamp[t] == cur) chp[A.posof[t] + 1]++;
    }
    for (int32_t q = 0; q < pn; q++) chp[q + 1] += chp[q];
    for (int32_t q = 0; q < pn; q++) fill[q] = chp[q];
    for (int32_t q = 0; q < pn; q++) {   // ascending members: ascending children per parent
        const int32_t x = mem[q], t = A.a[x];
        if (t != x && A.stamp[t] == cur) chl[fill[A.posof[t]]++] = x;
    }
}

// _detach_gain (detector.py:178-194) for sorted b (in_b marked)
__device__ double detach_gain(const LitArgs &A, const int32_t *b, int32_t nb, int64_t cur,
                              double so_c, double si_c, double *ws, double *tmp) {
    double x_w = 0.0;
    for (int32_t q = 0; q < nb; q++) {
        const int32_t y = b[q];
        int32_t cnt = 0;
        bool any = false;
        for (int64_t e = A.uptr[y]; e < A.uptr[y + 1]; e++) {
            const int32_t z = A.unbr[e];
            if (A.stamp[z] != cur) continue;
            any = true;
            if (!A.in_b[z]) ws[cnt++] = A.uu[e];
        }
        if (any) x_w += pw_sum_seq(ws, cnt);
    }
    const double so_b = gather_sum(A.s_out, b, nb, tmp), si_b = gather_sum(A.s_in, b, nb, tmp);
    const double null = (-so_c * si_b - so_b * si_c) + 2.0 * so_b * si_b;
    return -x_w / A.m - null / (A.m * A.m);
}

__global__ void k_positive_lit(LitArgs A, const LitJob *jobs, int32_t *ipool, double *dpool,
                               double *gains, LitOut *out, int64_t maxdeg) {
    if (threadIdx.x != 0) return;
    const LitJob J = jobs[blockIdx.x];
    const int32_t k = J.k;
    // int pool: parts (k), tmp (k), stack (2k), chp (k+1), chl (k), fill (k), sub (k),
    // best (k), cyc (k), path (k), grp (k), goff (k+1)
    int32_t *pool = ipool + J.ip, *tmpi = pool + k, *stk = tmpi + k, *chp = stk + 2 * k,
            *chl = chp + k + 1, *fill = chl + k, *sub = fill + k, *best = sub + k,
            *cyc = best + k, *path = cyc + k, *grp = path + k, *goff = grp + k;
    // double pool: gv (k), tmp (max(k, maxdeg)), ws (maxdeg), wsi (maxdeg), so_g (k), si_g (k)
    const int64_t tw = max((int64_t)k, maxdeg);
    double *gv = dpool + J.dp, *tmp = gv + k, *ws = tmp + tw, *wsi = ws + maxdeg,
           *so_g = wsi + maxdeg, *si_g = so_g + k;
    double *gout = gains + J.gp;
    LitOut o{0, 0, 0, 0};
    for (int32_t q = 0; q < k; q++) pool[q] = A.members[J.moff + q];
    int32_t sn = 0;
    stk[0] = 0;
    stk[1] = k;
    sn = 1;
    int64_t cur = ((int64_t)(blockIdx.x + 1) << 32);
    const double m = A.m, m2 = A.m2;
    while (sn > 0) {
        sn--;
        const int32_t off = stk[2 * sn], pn = stk[2 * sn + 1];
        int32_t *mem = pool + off;
        if (pn <= 1) continue;
        cur++;
        for (int32_t q = 0; q < pn; q++) {
            A.stamp[mem[q]] = cur;
            A.posof[mem[q]] = q;
        }
        const double so_c = gather_sum(A.s_out, mem, pn, tmp);
        const double si_c = gather_sum(A.s_in, mem, pn, tmp);
        bool any_neg = false;
        for (int32_t q = 0; q < pn; q++) {
            const int32_t x = mem[q];
            int32_t cnt = 0;
            for (int64_t e = A.uptr[x]; e < A.uptr[x + 1]; e++)
                if (A.stamp[A.unbr[e]] == cur) ws[cnt++] = A.uu[e];
            const double w_in_c = pw_sum_seq(ws, cnt);
            const double so = A.s_out[x], si = A.s_in[x];
            gv[q] = w_in_c / m - (so * (si_c - si) + si * (so_c - so)) / m2;
            any_neg |= gv[q] < 0.0;
        }
        if (!any_neg) continue;
        // _find_cycle from the smallest member (detector.py:163-175)
        int32_t plen = 0, x = mem[0];
        while (A.seen[x] < 0) {
            A.seen[x] = plen;
            path[plen++] = x;
            x = A.a[x];
        }
        const int32_t p0 = A.seen[x], s = plen - p0;
        int32_t kmin = p0;
        for (int32_t p = p0; p < plen; p++)
            if (path[p] < path[kmin]) kmin = p;
        for (int32_t q = 0; q < s; q++) cyc[q] = path[p0 + (kmin - p0 + q) % s];
        for (int32_t p = 0; p < plen; p++) A.seen[path[p]] = -1;
        part_children(A, mem, pn, cur, chp, chl, fill);
        // cycle membership by position (tmpi as a flag array)
        for (int32_t q = 0; q < pn; q++) tmpi[q] = 0;
        for (int32_t q = 0; q < s; q++) tmpi[A.posof[cyc[q]]] = 1;
        double best_gain = 0.0;
        int32_t bn = -1, cut0 = -1, cut1 = -1;
        // branch cuts (detector.py:238-253)
        for (int32_t q = 0; q < pn; q++) {
            if (tmpi[q]) continue;
            int32_t ns = 0;
            sub[ns++] = mem[q];
            for (int32_t qi = 0; qi < ns; qi++) {
                const int32_t py = A.posof[sub[qi]];
                for (int32_t c = chp[py]; c < chp[py + 1]; c++) sub[ns++] = chl[c];
            }
            heapsort_i32(sub, ns);
            for (int32_t t = 0; t < ns; t++) A.in_b[sub[t]] = 1;
            const double g = detach_gain(A, sub, ns, cur, so_c, si_c, ws, tmp);
            for (int32_t t = 0; t < ns; t++) A.in_b[sub[t]] = 0;
            if (g > best_gain) {
                best_gain = g;
                for (int32_t t = 0; t < ns; t++) best[t] = sub[t];
                bn = ns;
                cut0 = mem[q];
                cut1 = -1;
            }
        }
        if (bn < 0 && s >= 2) {
            if (s > A.scc_cap) {
                // peel the worst negative cycle node (detector.py:255-268)
                int32_t worst = -1;
                double wg = 0.0;
                for (int32_t q = 0; q < s; q++) {
                    const int32_t y = cyc[q];
                    const double gy = gv[A.posof[y]];
                    if (gy < 0.0 && (worst < 0 || gy < wg || (gy == wg && y < worst))) {
                        worst = y;
                        wg = gy;
                    }
                }
                if (worst >= 0) {
                    A.a[worst] = worst;
                    o.changed = 1;
                    o.nwarn++;
                    stk[2 * sn] = off;   // retry the same part
                    stk[2 * sn + 1] = pn;
                    sn++;
                    continue;
                }
            } else {
                // _best_pair_cut (detector.py:288-335): groups = cycle node + hanging subtrees
                int32_t gl = 0;
                for (int32_t q = 0; q < s; q++) {
                    goff[q] = gl;
                    int32_t *g = grp + gl;
                    int32_t ng = 0;
                    g[ng++] = cyc[q];
                    for (int32_t qi = 0; qi < ng; qi++) {
                        const int32_t py = A.posof[g[qi]];
                        for (int32_t c = chp[py]; c < chp[py + 1]; c++)
                            if (!tmpi[A.posof[chl[c]]]) g[ng++] = chl[c];
                    }
                    heapsort_i32(g, ng);
                    so_g[q] = gather_sum(A.s_out, g, ng, tmp);
                    si_g[q] = gather_sum(A.s_in, g, ng, tmp);
                    gl += ng;
                }
                goff[s] = gl;
                double pbest = 0.0;
                int32_t bp = -1, bq = -1;
                for (int32_t p = 0; p < s - 1; p++) {
                    for (int32_t t = 0; t < pn; t++) A.in_b[mem[t]] = 0;
                    double so_b = 0.0, si_b = 0.0, x_w = 0.0;
                    for (int32_t q = p + 1; q < s; q++) {
                        for (int32_t t = goff[q]; t < goff[q + 1]; t++) {
                            const int32_t y = grp[t];
                            int32_t c1 = 0, c2 = 0;
                            bool any = false;
                            for (int64_t e = A.uptr[y]; e < A.uptr[y + 1]; e++) {
                                const int32_t z = A.unbr[e];
                                if (A.stamp[z] != cur) continue;
                                any = true;
                                if (A.in_b[z]) wsi[c2++] = A.uu[e];
                                else ws[c1++] = A.uu[e];
                            }
                            if (any) x_w += pw_sum_seq(ws, c1) - pw_sum_seq(wsi, c2);
                            A.in_b[y] = 1;
                        }
                        so_b += so_g[q];
                        si_b += si_g[q];
                        const double null = (-so_c * si_b - so_b * si_c) + 2.0 * so_b * si_b;
                        const double gain = -x_w / m - null / m2;
                        if (gain > pbest) {
                            pbest = gain;
                            bp = p;
                            bq = q;
                        }
                    }
                }
                for (int32_t t = 0; t < pn; t++) A.in_b[mem[t]] = 0;
                if (bp >= 0 && pbest > best_gain) {
                    best_gain = pbest;
                    bn = 0;
                    for (int32_t t = goff[bp + 1]; t < goff[bq + 1]; t++) best[bn++] = grp[t];
                    heapsort_i32(best, bn);
                    cut0 = cyc[bp];
                    cut1 = cyc[bq];
                }
            }
        }
        if (bn < 0) {
            for (int32_t q = 0; q < pn; q++) o.unresolved += gv[q] < 0.0;
            continue;
        }
        A.a[cut0] = cut0;
        if (cut1 >= 0) A.a[cut1] = cut1;
        o.changed = 1;
        gout[o.ngains++] = best_gain;
        // rest = mem minus best (both sorted), then best: the part's slot holds [rest, best]
        int32_t rn = 0, bi = 0;
        for (int32_t q = 0; q < pn; q++) {
            while (bi < bn && best[bi] < mem[q]) bi++;
            if (bi < bn && best[bi] == mem[q]) continue;
            tmpi[rn++] = mem[q];
        }
        for (int32_t q = 0; q < rn; q++) mem[q] = tmpi[q];
        for (int32_t q = 0; q < bn; q++) mem[rn + q] = best[q];
        stk[2 * sn] = off;
        stk[2 * sn + 1] = rn;
        stk[2 * sn + 2] = off + rn;
        stk[2 * sn + 3] = bn;
        sn += 2;
    }
    out[blockIdx.x] = o;
}

// a node on a cycle longer than 2: on_cycle, not self-assigned, and its target's target is
// not itself; marks the node's community (and a global flag)
__global__ void k_long_cycle_marks(const int32_t *a, const uint8_t *on_cycle, const int32_t *comm,
                                   int64_t n, uint8_t *cflag, int32_t *any_long) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        if (!on_cycle[x]) continue;
        const int32_t t = a[x];
        if (t != (int32_t)x && a[t] != (int32_t)x) {
            cflag[comm[x]] = 1;
            *any_long = 1;
        }
    }
}
__global__ void k_bad_long(const int32_t *list, int32_t nbad, const uint8_t *cflag, int32_t *len) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nbad;
         i += (int64_t)gridDim.x * blockDim.x)
        len[i] = cflag[list[i]] ? 3 : 0;
}

}  // namespace

// per bad community: > 2 when its assignment cycle is longer than 2 (else 0); one O(n)
// pass over the forest, and nothing more is read back unless such a cycle exists
void bad_cycle_lengths(slm_ctx *ctx, const Forest &F, const int32_t *d_list, int32_t nbad,
                       std::vector<int32_t> &h_len) {
    cudaStream_t s = ctx->stream;
    h_len.assign(nbad, 0);
    if (!nbad || F.n == 0) return;
    DBuf<int32_t> any;
    any.resize(1);
    CTX_SCRATCH(DBuf<uint8_t>, cflag);
    cflag.resize(F.n_comms);
    CUDA_TRY(cudaMemsetAsync(any.p, 0, 4, s));
    CUDA_TRY(cudaMemsetAsync(cflag.p, 0, F.n_comms, s));
    k_long_cycle_marks<<<grid_for(F.n, 256), 256, 0, s>>>(F.a.p, F.on_cycle.p, F.comm.p, F.n,
                                                         cflag.p, any.p);
    int32_t h_any = 0;
    CUDA_TRY(cudaMemcpyAsync(&h_any, any.p, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (!h_any) return;
    DBuf<int32_t> d;
    d.resize(nbad);
    k_bad_long<<<grid_for(nbad, 256), 256, 0, s>>>(d_list, nbad, cflag.p, d.p);
    CUDA_TRY(cudaMemcpyAsync(h_len.data(), d.p, nbad * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
}

// POSITIVE for the given communities (community ids + member ranges), literal algorithm;
// per community: gains in the reference's order, splits, unresolved, changed flag
void run_positive_literal(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m,
                          int64_t scc_cap, const std::vector<int2> &ranges,
                          std::vector<std::vector<double>> &gains, std::vector<int32_t> &unres,
                          std::vector<int32_t> &changed, int64_t *nwarn) {
    cudaStream_t s = ctx->stream;
    const int32_t nj = (int32_t)ranges.size();
    gains.assign(nj, {});
    unres.assign(nj, 0);
    changed.assign(nj, 0);
    *nwarn = 0;
    if (!nj) return;
    // the largest union row among the jobs' members sizes the per-row scratch
    std::vector<LitJob> jobs(nj);
    int64_t ip = 0, dp = 0, gp = 0;
    int64_t maxdeg = 1;
    {
        std::vector<int32_t> hm(G.n);
        std::vector<int64_t> up(G.n + 1);
        CUDA_TRY(cudaMemcpyAsync(up.data(), G.uptr.p, (G.n + 1) * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(hm.data(), F.members.p, G.n * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        for (const int2 &r : ranges)
            for (int32_t q = r.x; q < r.y; q++)
                maxdeg = std::max<int64_t>(maxdeg, up[hm[q] + 1] - up[hm[q]]);
    }
    for (int32_t j = 0; j < nj; j++) {
        const int32_t k = ranges[j].y - ranges[j].x;
        jobs[j] = LitJob{ranges[j].x, k, ip, dp, gp};
        ip += 14 * (int64_t)k + 4;
        dp += 4 * (int64_t)k + std::max<int64_t>(k, maxdeg) + 2 * maxdeg;
        gp += k;
    }
    DBuf<LitJob> dj;
    DBuf<int32_t> ipool, seen, posof;
    DBuf<double> dpool, gbuf;
    DBuf<int64_t> stamp;
    DBuf<uint8_t> inb;
    DBuf<LitOut> dout;
    dj.resize(nj);
    ipool.resize(ip);
    dpool.resize(dp);
    gbuf.resize(std::max<int64_t>(1, gp));
    stamp.resize(G.n);
    inb.resize(G.n);
    seen.resize(G.n);
    posof.resize(G.n);
    dout.resize(nj);
    CUDA_TRY(cudaMemcpyAsync(dj.p, jobs.data(), nj * sizeof(LitJob), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(stamp.p, 0, G.n * 8, s));
    CUDA_TRY(cudaMemsetAsync(inb.p, 0, G.n, s));
    CUDA_TRY(cudaMemsetAsync(seen.p, 0xff, G.n * 4, s));
    LitArgs A{G.uptr.p, G.unbr.p, G.uu.p, G.s_out.p, G.s_in.p, F.a.p, m, m * m, scc_cap,
              stamp.p, inb.p, seen.p, posof.p, F.members.p};
    k_positive_lit<<<nj, 32, 0, s>>>(A, dj.p, ipool.p, dpool.p, gbuf.p, dout.p, maxdeg);
    CUDA_TRY(cudaGetLastError());
    std::vector<LitOut> ho(nj);
    std::vector<double> hg(std::max<int64_t>(1, gp));
    CUDA_TRY(cudaMemcpyAsync(ho.data(), dout.p, nj * sizeof(LitOut), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(hg.data(), gbuf.p, std::max<int64_t>(1, gp) * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int32_t j = 0; j < nj; j++) {
        gains[j].assign(hg.begin() + jobs[j].gp, hg.begin() + jobs[j].gp + ho[j].ngains);
        unres[j] = ho[j].unresolved;
        changed[j] = ho[j].changed;
        *nwarn += ho[j].nwarn;
    }
}

const void *slm_anchor_positive_lit() { return (const void *)k_positive_lit; }
