// slm_level.cu -- AGGREGATE (aggregate, graph.py:266-280) and SCORE (score, quality.py:104-118).
//
// Aggregation is Graph.from_edges over (label[src], label[dst], w) in CSR order, i.e. the
// same packed-key radix sort + run merge as the level-0 build, so intra-community weight
// becomes self-loops and m_w is preserved.  The score keeps numpy's evaluation order:
// intra = pairwise sum of the masked CSR weights (CSR order), S per community by
// sequential sums in node order, null = pairwise sum of S_out*S_in/m over communities.
#include "slm_internal.cuh"

#define GS_LOOP(i, n)                                                                      \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n);              \
         i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_coarse_keys(const int64_t *ptr, const int32_t *dst, const double *w,
                              const int32_t *lab, int64_t n, int b, uint64_t *keys, double *vals) {
    const int lane = threadIdx.x & 31;
    int64_t wi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = wi; r < n; r += nw) {
        const uint64_t cs = (uint64_t)(uint32_t)lab[r] << b;
        for (int64_t e = ptr[r] + lane; e < ptr[r + 1]; e += 32) {
            keys[e] = cs | (uint32_t)lab[dst[e]];
            vals[e] = w[e];
        }
    }
}

void run_aggregate(slm_ctx *ctx, const LevelGraph &G, const int32_t *d_labels, int64_t n_comms,
                   LevelGraph &out) {
    CTX_SCRATCH(DBuf<uint64_t>, keys);   // grow-only scratch kept across levels
    CTX_SCRATCH(DBuf<double>, vals);
    keys.resize(G.ne);
    vals.resize(G.ne);
    if (G.ne > 0)
        k_coarse_keys<<<grid_for(G.n * 32, 256, SMS() * 64), 256, 0, ctx->stream>>>(
            G.csr_ptr.p, G.csr_dst.p, G.csr_w.p, d_labels, G.n, bits_for(n_comms), keys.p, vals.p);
    build_level_from_keys(ctx, out, n_comms, keys, vals, G.ne);
}

__global__ void k_intra_flags(const int64_t *ptr, const int32_t *dst, const int32_t *lab,
                              int64_t n, int64_t *flag) {
    const int lane = threadIdx.x & 31;
    int64_t wi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = wi; r < n; r += nw) {
        const int32_t L = lab[r];
        for (int64_t e = ptr[r] + lane; e < ptr[r + 1]; e += 32) flag[e] = (lab[dst[e]] == L);
    }
}
__global__ void k_compact_f64(const double *v, const int64_t *flag, const int64_t *pos, int64_t m,
                              double *out) {
    GS_LOOP(e, m) if (flag[e]) out[pos[e]] = v[e];
}
__global__ void k_max_i32(const int32_t *x, int64_t n, int32_t *mx, int32_t *mn) {
    int32_t a = INT32_MIN, b = INT32_MAX;
    GS_LOOP(i, n) {
        a = max(a, x[i]);
        b = min(b, x[i]);
    }
    a = __reduce_max_sync(0xffffffffu, a);   // one atomic pair per warp
    b = __reduce_min_sync(0xffffffffu, b);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(mx, a);
        atomicMin(mn, b);
    }
}
__global__ void k_null_terms(const double *So, const double *Si, int64_t nc, double m, double *out) {
    GS_LOOP(c, nc) out[c] = So[c] * Si[c] / m;
}
__global__ void k_iota32(int32_t *x, int64_t n) { GS_LOOP(i, n) x[i] = (int32_t)i; }
__global__ void k_lb32(const int32_t *sorted, int64_t m, int64_t nrows, int32_t *ptr) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= nrows;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = m;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (sorted[mid] < r) lo = mid + 1;
            else hi = mid;
        }
        ptr[r] = (int32_t)lo;
    }
}
__global__ void k_seg_seq_sums(const int32_t *cptr, const int32_t *members, const double *a,
                               const double *b, int64_t nc, double *A, double *B) {
    GS_LOOP(c, nc) {
        double x = 0.0, y = 0.0;
        for (int32_t k = cptr[c]; k < cptr[c + 1]; k++) {
            x += a[members[k]];
            y += b[members[k]];
        }
        A[c] = x;
        B[c] = y;
    }
}

double run_score(slm_ctx *ctx, const LevelGraph &G, const int32_t *d_labels, double gamma) {
    cudaStream_t s = ctx->stream;
    const double m = G.m_w;
    if (m == 0.0 || G.n == 0) return 0.0;
    const int64_t n = G.n, ne = G.ne;
    // intra: masked out_w in CSR order, pairwise (quality.py:113)
    DBuf<int64_t> flag, pos;
    DBuf<double> comp;
    flag.resize(ne + 1);
    pos.resize(ne + 1);
    CUDA_TRY(cudaMemsetAsync(flag.p + ne, 0, 8, s));
    k_intra_flags<<<grid_for(n * 32, 256, SMS() * 64), 256, 0, s>>>(G.csr_ptr.p, G.csr_dst.p,
                                                                     d_labels, n, flag.p);
    dev_exclusive_sum<int64_t, int64_t>(ctx, flag.p, pos.p, ne + 1);
    int64_t nin = 0;
    CUDA_TRY(cudaMemcpyAsync(&nin, pos.p + ne, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    comp.resize(nin);
    k_compact_f64<<<grid_for(ne, 256), 256, 0, s>>>(G.csr_w.p, flag.p, pos.p, ne, comp.p);
    double intra = device_pairwise_sum(ctx, comp.p, nin);
    flag.release();
    pos.release();
    comp.release();
    // communities 0..max(label) (quality.py:114-117)
    int32_t *mm = ctx->i32d.resize(2);
    int32_t init[2] = {-1, 0x7fffffff};
    CUDA_TRY(cudaMemcpyAsync(mm, init, 8, cudaMemcpyHostToDevice, s));
    k_max_i32<<<grid_for(n, 256), 256, 0, s>>>(d_labels, n, mm, mm + 1);
    int32_t hm[2];
    CUDA_TRY(cudaMemcpyAsync(hm, mm, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    SLM_REQUIRE(hm[1] >= 0, SLM_EINVAL, "labels must be non-negative");
    const int64_t nc = (int64_t)hm[0] + 1;
    DBuf<int32_t> iota, members, ksorted, cptr;
    DBuf<double> So, Si, terms;
    iota.resize(n);
    members.resize(n);
    ksorted.resize(n);
    cptr.resize(nc + 1);
    k_iota32<<<grid_for(n, 256), 256, 0, s>>>(iota.p, n);
    sort_pairs_u32_i32(ctx, (uint32_t *)d_labels, (uint32_t *)ksorted.p, iota.p, members.p, n,
                       bits_for(nc + 1));
    k_lb32<<<grid_for(nc + 1, 256), 256, 0, s>>>(ksorted.p, n, nc, cptr.p);
    So.resize(nc);
    Si.resize(nc);
    terms.resize(nc);
    k_seg_seq_sums<<<grid_for(nc, 128), 128, 0, s>>>(cptr.p, members.p, G.s_out.p, G.s_in.p, nc,
                                                     So.p, Si.p);
    k_null_terms<<<grid_for(nc, 256), 256, 0, s>>>(So.p, Si.p, nc, m, terms.p);
    double null = device_pairwise_sum(ctx, terms.p, nc);
    return (intra - gamma * null) / m;
}

// a kernel of this translation unit (module preloading, slm_capi.cu preload_modules)
const void *slm_anchor_level() { return (const void *)k_coarse_keys; }
