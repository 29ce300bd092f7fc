// slm_surface.cu -- the rest of the reference's hot-path API surface on the device:
//   CommunityAggregates.from_labels   quality.py:71-79   sequential per-community sums
//   gain_switch                       quality.py:186-219 exact score change of a set move
//   reverse_assignment                forest.py:70-80    children CSR of the assignment map
//   NeighborUnion.w_out / w_in        graph.py:46-60     split of the pre-summed union weight
//   canonicalize_labels               graph.py:283-291   dense labels by first occurrence
// (aggregate, graph.py:266-280, reuses the level build: run_aggregate in slm_level.cu).
// Every fp64 sum keeps the reference's order (bincount: sequential in node order; ndarray
// .sum(): numpy pairwise), so the results are bit-identical for real-valued weights too.
#include "slm_internal.cuh"

#define GS_LOOP(i, n)                                                                      \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n);              \
         i += (int64_t)gridDim.x * blockDim.x)

namespace {

__global__ void k_iota(int32_t *x, int64_t n) { GS_LOOP(i, n) x[i] = (int32_t)i; }
__global__ void k_count(const int32_t *lab, int64_t n, int32_t *cnt) {
    GS_LOOP(i, n) atomicAdd(cnt + lab[i], 1);
}
// per community, sequential sums over its members in ascending node order (np.bincount)
__global__ void k_comm_sums(const int32_t *members, const int32_t *cptr, int64_t nc,
                            const double *s_out, const double *s_in, double *S_out, double *S_in) {
    GS_LOOP(c, nc) {
        double a = 0.0, b = 0.0;
        for (int32_t k = cptr[c]; k < cptr[c + 1]; k++) {
            const int32_t x = members[k];
            a += s_out[x];
            b += s_in[x];
        }
        S_out[c] = a;
        S_in[c] = b;
    }
}

// gain_switch: per moved node, the entries of its union row whose neighbour is in `to`
// (w_to) or in `frm` and not moved (w_from); counted, then written compactly in row order
__global__ void k_gs_count(const int64_t *uptr, const int32_t *unbr, const int32_t *lab,
                           const uint8_t *inset, const int32_t *nodes, int64_t k, int32_t frm,
                           int32_t to, int64_t *cto, int64_t *cfr) {
    GS_LOOP(q, k) {
        const int32_t x = nodes[q];
        int64_t a = 0, b = 0;
        for (int64_t e = uptr[x]; e < uptr[x + 1]; e++) {
            const int32_t z = unbr[e], l = lab[z];
            a += (to >= 0 && l == to);
            b += (l == frm && !inset[z]);
        }
        cto[q] = a;
        cfr[q] = b;
    }
}
__global__ void k_gs_fill(const int64_t *uptr, const int32_t *unbr, const double *uu,
                          const int32_t *lab, const uint8_t *inset, const int32_t *nodes, int64_t k,
                          int32_t frm, int32_t to, const int64_t *oto, const int64_t *ofr,
                          double *vto, double *vfr) {
    GS_LOOP(q, k) {
        const int32_t x = nodes[q];
        int64_t a = oto[q], b = ofr[q];
        for (int64_t e = uptr[x]; e < uptr[x + 1]; e++) {
            const int32_t z = unbr[e], l = lab[z];
            if (to >= 0 && l == to) vto[a++] = uu[e];
            if (l == frm && !inset[z]) vfr[b++] = uu[e];
        }
    }
}
__global__ void k_gs_rowsums(const int64_t *oto, const int64_t *ofr, const double *vto,
                             const double *vfr, int64_t k, double *wto, double *wfr) {
    GS_LOOP(q, k) {
        wto[q] = pw_sum_seq(vto + oto[q], oto[q + 1] - oto[q]);
        wfr[q] = pw_sum_seq(vfr + ofr[q], ofr[q + 1] - ofr[q]);
    }
}
// one thread: the reference's accumulation order and fp64 expression (quality.py:205-219)
__global__ void k_gs_final(const double *wto, const double *wfr, const int32_t *nodes, int64_t k,
                           const double *s_out, const double *s_in, double *gso, double *gsi,
                           double4 agg, int has_to, double m, double *gain) {
    double w_to = 0.0, w_from = 0.0;
    for (int64_t q = 0; q < k; q++) {
        if (has_to) w_to += wto[q];
        w_from += wfr[q];
        gso[q] = s_out[nodes[q]];
        gsi[q] = s_in[nodes[q]];
    }
    const double so_b = pw_sum_seq(gso, k), si_b = pw_sum_seq(gsi, k);
    const double so_t = has_to ? agg.z : 0.0, si_t = has_to ? agg.w : 0.0;
    const double d_null = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(
        __dmul_rn(-agg.x, si_b), -__dmul_rn(so_b, agg.y)), __dmul_rn(so_t, si_b)),
        __dmul_rn(so_b, si_t)), __dmul_rn(__dmul_rn(2.0, so_b), si_b));
    *gain = __dadd_rn(__ddiv_rn(__dadd_rn(w_to, -w_from), m),
                      -__ddiv_rn(d_null, __dmul_rn(m, m)));
}

__global__ void k_rev_keys(const int32_t *a, int64_t n, uint32_t *key, int32_t *cnt) {
    GS_LOOP(j, n) {
        const int32_t t = a[j];
        if (t != (int32_t)j) {
            key[j] = (uint32_t)t;
            atomicAdd(cnt + t, 1);
        } else {
            key[j] = (uint32_t)n;   // self-assigned: sorts after every target
        }
    }
}

// w_out[e] = W(i, j), w_in[e] = W(j, i) (0.0 when absent) for union entry e = (i, j):
// binary searches in the ascending CSR rows of i and j; one warp per row
__device__ __forceinline__ double csr_weight(const int64_t *ptr, const int32_t *dst,
                                             const double *w, int32_t i, int32_t j) {
    int64_t lo = ptr[i], hi = ptr[i + 1];
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (dst[mid] < j) lo = mid + 1;
        else hi = mid;
    }
    return (lo < ptr[i + 1] && dst[lo] == j) ? w[lo] : 0.0;
}
__global__ void k_union_split(const int64_t *uptr, const int32_t *unbr, const int64_t *cptr,
                              const int32_t *cdst, const double *cw, int64_t n, double *wo,
                              double *wi) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w0; i < n; i += nw)
        for (int64_t e = uptr[i] + lane; e < uptr[i + 1]; e += 32) {
            const int32_t j = unbr[e];
            wo[e] = __dadd_rn(csr_weight(cptr, cdst, cw, (int32_t)i, j), 0.0);
            wi[e] = __dadd_rn(0.0, csr_weight(cptr, cdst, cw, j, (int32_t)i));
        }
}

// canonicalize: label of the node at sorted position p is a run head when it differs from
// its predecessor; the run's first node (stable sort) is its first occurrence
__global__ void k_canon_heads(const uint32_t *ks, const int32_t *vs, int64_t n, uint32_t *first,
                              int32_t *rank_of_node_run) {
    GS_LOOP(p, n) {
        const bool head = p == 0 || ks[p] != ks[p - 1];
        rank_of_node_run[p] = head ? 1 : 0;
        if (head) first[p] = (uint32_t)vs[p];
    }
}

__global__ void k_set_flags(uint8_t *f, const int32_t *x, int64_t k) { GS_LOOP(q, k) f[x[q]] = 1; }
__global__ void k_canon_compact(const uint32_t *first, const int32_t *head, const int32_t *hpos,
                                int64_t n, uint32_t *fs) {
    GS_LOOP(p, n) if (head[p]) fs[hpos[p]] = first[p];
}
__global__ void k_canon_rank(const int32_t *gsorted, int64_t nu, int32_t *rk) {
    GS_LOOP(r, nu) rk[gsorted[r]] = (int32_t)r;
}
// group of sorted position p = (inclusive head count at p) - 1 = hpos[p] + head[p] - 1
__global__ void k_canon_scatter(const int32_t *vs, const int32_t *head, const int32_t *hpos,
                                const int32_t *rk, int64_t n, int32_t *out) {
    GS_LOOP(p, n) out[vs[p]] = rk[hpos[p] + head[p] - 1];
}

}  // namespace

void comm_sums_device(slm_ctx *ctx, const int32_t *d_lab, int64_t n, int64_t nc,
                      const double *d_so, const double *d_si, double *d_So, double *d_Si,
                      int32_t *d_cnt) {
    cudaStream_t s = ctx->stream;
    DBuf<int32_t> iota, members, cptr, cnt;
    DBuf<uint32_t> ks;
    iota.resize(n);
    members.resize(n);
    ks.resize(n);
    cnt.resize(nc + 1);
    cptr.resize(nc + 1);
    CUDA_TRY(cudaMemsetAsync(cnt.p, 0, (nc + 1) * 4, s));
    if (n) {
        k_iota<<<grid_for(n, 256), 256, 0, s>>>(iota.p, n);
        k_count<<<grid_for(n, 256), 256, 0, s>>>(d_lab, n, cnt.p);
        sort_pairs_u32_i32(ctx, (uint32_t *)d_lab, ks.p, iota.p, members.p, n, bits_for(nc + 1));
    }
    dev_exclusive_sum<int32_t, int32_t>(ctx, cnt.p, cptr.p, nc + 1);
    if (nc) {
        k_comm_sums<<<grid_for(nc, 128), 128, 0, s>>>(members.p, cptr.p, nc, d_so, d_si, d_So, d_Si);
        CUDA_TRY(cudaMemcpyAsync(d_cnt, cnt.p, nc * 4, cudaMemcpyDeviceToDevice, s));
    }
    CUDA_TRY(cudaGetLastError());
}

double gain_switch_device(slm_ctx *ctx, const LevelGraph &G, const int32_t *d_lab,
                          const int32_t *d_nodes, int64_t k, int32_t frm, int32_t to,
                          const double agg[4], double m) {
    cudaStream_t s = ctx->stream;
    DBuf<uint8_t> inset;
    DBuf<int64_t> cto, cfr, oto, ofr;
    DBuf<double> vto, vfr, wto, wfr, gso, gsi, g;
    inset.resize(G.n);
    CUDA_TRY(cudaMemsetAsync(inset.p, 0, G.n, s));
    cto.resize(k + 1);
    cfr.resize(k + 1);
    oto.resize(k + 1);
    ofr.resize(k + 1);
    wto.resize(k);
    wfr.resize(k);
    gso.resize(k);
    gsi.resize(k);
    g.resize(1);
    if (k) k_set_flags<<<grid_for(k, 256), 256, 0, s>>>(inset.p, d_nodes, k);
    CUDA_TRY(cudaMemsetAsync(cto.p + k, 0, 8, s));
    CUDA_TRY(cudaMemsetAsync(cfr.p + k, 0, 8, s));
    if (k)
        k_gs_count<<<grid_for(k, 128), 128, 0, s>>>(G.uptr.p, G.unbr.p, d_lab, inset.p, d_nodes, k,
                                                    frm, to, cto.p, cfr.p);
    dev_exclusive_sum<int64_t, int64_t>(ctx, cto.p, oto.p, k + 1);
    dev_exclusive_sum<int64_t, int64_t>(ctx, cfr.p, ofr.p, k + 1);
    int64_t tot[2] = {0, 0};
    CUDA_TRY(cudaMemcpyAsync(tot, oto.p + k, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(tot + 1, ofr.p + k, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    vto.resize(std::max<int64_t>(1, tot[0]));
    vfr.resize(std::max<int64_t>(1, tot[1]));
    if (k) {
        k_gs_fill<<<grid_for(k, 128), 128, 0, s>>>(G.uptr.p, G.unbr.p, G.uu.p, d_lab, inset.p,
                                                   d_nodes, k, frm, to, oto.p, ofr.p, vto.p, vfr.p);
        k_gs_rowsums<<<grid_for(k, 128), 128, 0, s>>>(oto.p, ofr.p, vto.p, vfr.p, k, wto.p, wfr.p);
    }
    k_gs_final<<<1, 1, 0, s>>>(wto.p, wfr.p, d_nodes, k, G.s_out.p, G.s_in.p, gso.p, gsi.p,
                               make_double4(agg[0], agg[1], agg[2], agg[3]), to >= 0 ? 1 : 0, m,
                               g.p);
    double out = 0.0;
    CUDA_TRY(cudaMemcpyAsync(&out, g.p, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return out;
}

void reverse_assignment_device(slm_ctx *ctx, const int32_t *d_a, int64_t n, int64_t *h_ptr,
                               int64_t *h_kids, int64_t *h_nk) {
    cudaStream_t s = ctx->stream;
    DBuf<uint32_t> key, ks;
    DBuf<int32_t> iota, kids, cnt, ptr32;
    key.resize(n);
    ks.resize(n);
    iota.resize(n);
    kids.resize(n);
    cnt.resize(n + 1);
    ptr32.resize(n + 1);
    CUDA_TRY(cudaMemsetAsync(cnt.p, 0, (n + 1) * 4, s));
    if (n) {
        k_rev_keys<<<grid_for(n, 256), 256, 0, s>>>(d_a, n, key.p, cnt.p);
        k_iota<<<grid_for(n, 256), 256, 0, s>>>(iota.p, n);
        sort_pairs_u32_i32(ctx, key.p, ks.p, iota.p, kids.p, n, bits_for(n + 1));
    }
    dev_exclusive_sum<int32_t, int32_t>(ctx, cnt.p, ptr32.p, n + 1);
    std::vector<int32_t> p(n + 1);
    CUDA_TRY(cudaMemcpyAsync(p.data(), ptr32.p, (n + 1) * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    const int64_t nk = p[n];
    std::vector<int32_t> kk(nk);
    if (nk) CUDA_TRY(cudaMemcpy(kk.data(), kids.p, nk * 4, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i <= n; i++) h_ptr[i] = p[i];
    if (h_kids)
        for (int64_t i = 0; i < nk; i++) h_kids[i] = kk[i];
    *h_nk = nk;
}

void union_split_device(slm_ctx *ctx, const LevelGraph &G, double *d_wo, double *d_wi) {
    if (G.ue == 0) return;
    k_union_split<<<grid_for(G.n * 32, 256), 256, 0, ctx->stream>>>(
        G.uptr.p, G.unbr.p, G.csr_ptr.p, G.csr_dst.p, G.csr_w.p, G.n, d_wo, d_wi);
    CUDA_TRY(cudaGetLastError());
}

// labels (values 0..vmax) -> dense labels ordered by first occurrence; returns the count
int64_t canonicalize_device(slm_ctx *ctx, const uint32_t *d_lab, int64_t n, int end_bit,
                            int32_t *d_out) {
    cudaStream_t s = ctx->stream;
    if (n == 0) return 0;
    DBuf<uint32_t> ks, first, fs;
    DBuf<int32_t> iota, vs, head, hpos, ord, rk;
    ks.resize(n);
    iota.resize(n);
    vs.resize(n);
    head.resize(n + 1);
    hpos.resize(n + 1);
    first.resize(n);
    k_iota<<<grid_for(n, 256), 256, 0, s>>>(iota.p, n);
    // nodes grouped by label, ascending node id inside a group (stable)
    sort_pairs_u32_i32(ctx, (uint32_t *)d_lab, ks.p, iota.p, vs.p, n, end_bit);
    CUDA_TRY(cudaMemsetAsync(head.p + n, 0, 4, s));
    k_canon_heads<<<grid_for(n, 256), 256, 0, s>>>(ks.p, vs.p, n, first.p, head.p);
    dev_exclusive_sum<int32_t, int32_t>(ctx, head.p, hpos.p, n + 1);
    int32_t nu = 0;
    CUDA_TRY(cudaMemcpyAsync(&nu, hpos.p + n, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    // groups (in label order) -> their first occurrence; sort groups by it -> rank
    fs.resize(nu);
    ord.resize(nu);
    rk.resize(nu);
    DBuf<uint32_t> fsorted;
    DBuf<int32_t> gid, gidsorted;
    fsorted.resize(nu);
    gid.resize(nu);
    gidsorted.resize(nu);
    k_canon_compact<<<grid_for(n, 256), 256, 0, s>>>(first.p, head.p, hpos.p, n, fs.p);
    k_iota<<<grid_for(nu, 256), 256, 0, s>>>(gid.p, nu);
    sort_pairs_u32_i32(ctx, fs.p, fsorted.p, gid.p, gidsorted.p, nu, bits_for(n + 1));
    k_canon_rank<<<grid_for(nu, 256), 256, 0, s>>>(gidsorted.p, nu, rk.p);
    k_canon_scatter<<<grid_for(n, 256), 256, 0, s>>>(vs.p, head.p, hpos.p, rk.p, n, d_out);
    CUDA_TRY(cudaGetLastError());
    return nu;
}

const void *slm_anchor_surface() { return (const void *)k_iota; }
