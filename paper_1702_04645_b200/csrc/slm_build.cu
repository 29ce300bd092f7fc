// slm_build.cu -- device CSR build (Graph.from_edges, graph.py:84-116), neighbour union
// (_build_union, graph.py:151-175), strengths (graph.py:257-263) and degree binning.
//
// Edge list -> packed 2b-bit keys (src << b | dst) -> stable LSD radix sort with the weights
// as values -> run-length merge (each run summed first + pairwise(rest), numpy's reduceat
// order, so even real-valued duplicates merge bit-identically) -> CSR.  The union of a
// symmetric graph is the CSR minus self-loops with u = w + w (no second sort); a directed
// graph merges its out-row with its in-row (stable transpose).
#include "slm_internal.cuh"
#include <algorithm>
#include <cstdlib>

int bits_for(int64_t v) {
    int b = 1;
    while ((int64_t(1) << b) < v) b++;
    return b;
}

// ------------------------------------------------------------------- kernels

__global__ void k_validate(const int32_t *src, const int32_t *dst, const double *w, int64_t ne,
                           int64_t n, int32_t *bad) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
         e += (int64_t)gridDim.x * blockDim.x) {
        int32_t s = src[e], d = dst[e];
        double x = w[e];
        if (s < 0 || d < 0 || s >= n || d >= n) atomicOr(bad, 1);
        if (!(x > 0.0) || !isfinite(x)) atomicOr(bad, 2);
    }
}

__global__ void k_make_keys(const int32_t *src, const int32_t *dst, const double *w, int64_t ne,
                            int b, uint64_t *keys, double *vals) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
         e += (int64_t)gridDim.x * blockDim.x) {
        keys[e] = ((uint64_t)(uint32_t)src[e] << b) | (uint32_t)dst[e];
        vals[e] = w[e];
    }
}

__global__ void k_run_heads(const uint64_t *keys, int64_t ne, int64_t *head) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
         e += (int64_t)gridDim.x * blockDim.x)
        head[e] = (e == 0 || keys[e] != keys[e - 1]) ? 1 : 0;
}

// one thread per run: out_w = first + pairwise(rest) (np.add.reduceat, graph.py:108)
// runs longer than this (an aggregated giant community's self-loop run can hold 10^8
// entries) are summed by device_pairwise_sum instead of one thread
constexpr int64_t LONG_RUN = 4096;
constexpr int32_t MAX_LONG = 1 << 20;

__global__ void k_merge_runs(const uint64_t *keys, const double *vals, const int64_t *gid,
                             int64_t ne, int b, int32_t *out_src, int32_t *out_dst, double *out_w,
                             uint32_t *integral_bad, int64_t *long_runs, int32_t *nlong) {
    const uint64_t mask = (b >= 64) ? ~0ull : ((1ull << b) - 1);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (!(e == 0 || keys[e] != keys[e - 1])) continue;
        int64_t end = e + 1;
        while (end < ne && end - e <= LONG_RUN && keys[end] == keys[e]) end++;
        int64_t g = gid[e];
        out_src[g] = (int32_t)(keys[e] >> b);
        out_dst[g] = (int32_t)(keys[e] & mask);
        if (end - e > LONG_RUN) {   // long run: summed (and its integrality checked) separately
            const int at = atomicAdd(nlong, 1);
            long_runs[2 * at] = e;
            long_runs[2 * at + 1] = g;
            continue;
        }
        double s = reduceat_seq(vals + e, end - e);
        out_w[g] = s;
        for (int64_t q = e; q < end; q++)
            if (vals[q] != floor(vals[q])) atomicOr(integral_bad, 1u);
    }
}
// ptr[r] = first index i with key_of(i) >= r over a sorted int32 array (n_rows + 1 entries)
__global__ void k_lower_bound_ptr(const int32_t *sorted_rows, int64_t m, int64_t n_rows,
                                  int64_t *ptr) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = m;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (sorted_rows[mid] < r) lo = mid + 1;
            else hi = mid;
        }
        ptr[r] = lo;
    }
}

__global__ void k_iota_i32(int32_t *x, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = (int32_t)i;
}

__global__ void k_gather_transpose(const int32_t *perm, const int32_t *src, const double *w,
                                   int64_t ne, int32_t *in_src, double *in_w) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < ne;
         p += (int64_t)gridDim.x * blockDim.x) {
        int32_t e = perm[p];
        in_src[p] = src[e];
        in_w[p] = w[e];
    }
}

__global__ void k_sym_check(const int64_t *optr, const int32_t *odst, const double *ow,
                            const int64_t *iptr, const int32_t *isrc, const double *iw, int64_t n,
                            int64_t ne, int32_t *asym) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = t; i <= n; i += stride)
        if (optr[i] != iptr[i]) atomicOr(asym, 1);
    for (int64_t e = t; e < ne; e += stride)
        if (odst[e] != isrc[e] || ow[e] != iw[e]) atomicOr(asym, 1);
}

// symmetric graph: union = CSR minus self loops, u = w + w
__global__ void k_keep_nonself(const int64_t *ptr, const int32_t *dst, int64_t n, int64_t *keep) {
    // one warp per row
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int lane = threadIdx.x & 31;
    for (int64_t r = warp; r < n; r += nw)
        for (int64_t e = ptr[r] + lane; e < ptr[r + 1]; e += 32) keep[e] = (dst[e] != r) ? 1 : 0;
}

__global__ void k_fill_union_sym(const int64_t *ptr, const int32_t *dst, const double *w,
                                 const int64_t *pos, int64_t n, int64_t ne, int64_t ue,
                                 int64_t *uptr, int32_t *unbr, double *uu) {
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int lane = threadIdx.x & 31;
    for (int64_t r = warp; r < n; r += nw) {
        if (lane == 0) uptr[r] = (ptr[r] < ne) ? pos[ptr[r]] : ue;
        for (int64_t e = ptr[r] + lane; e < ptr[r + 1]; e += 32)
            if (dst[e] != r) {
                int64_t q = pos[e];
                unbr[q] = dst[e];
                uu[q] = w[e] + w[e];
            }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) uptr[n] = ue;
}

// directed graph: per-row merge of the out-row and the in-row (both sorted), self excluded.
// pass 0 counts, pass 1 fills.  u = W(i,j) + W(j,i) with absent directions contributing
// nothing (the reference's +0.0 is exact).
__global__ void k_union_merge(const int64_t *optr, const int32_t *odst, const double *ow,
                              const int64_t *iptr, const int32_t *isrc, const double *iw,
                              int64_t n, int pass, int64_t *cnt_or_uptr, int32_t *unbr,
                              double *uu) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = optr[r], ae = optr[r + 1], b = iptr[r], be = iptr[r + 1];
        int64_t k = pass ? cnt_or_uptr[r] : 0;
        for (;;) {
            while (a < ae && odst[a] == r) a++;
            while (b < be && isrc[b] == r) b++;
            if (a >= ae && b >= be) break;
            int32_t j;
            double u;
            if (b >= be || (a < ae && odst[a] < isrc[b])) {
                j = odst[a]; u = ow[a]; a++;
            } else if (a >= ae || isrc[b] < odst[a]) {
                j = isrc[b]; u = iw[b]; b++;
            } else {
                j = odst[a]; u = ow[a] + iw[b]; a++; b++;
            }
            if (pass) { unbr[k] = j; uu[k] = u; }
            k++;
        }
        if (!pass) cnt_or_uptr[r] = k;
    }
}

// bincount order: sequential per row (graph.py:258-259)
__global__ void k_row_seq_sum(const int64_t *ptr, const double *w, int64_t n, double *out) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t e = ptr[r]; e < ptr[r + 1]; e++) s += w[e];
        out[r] = s;
    }
}

__global__ void k_pw_segments(const double *a, const int64_t *off, const int64_t *len, int64_t k,
                              double *out, uint32_t *nonint = nullptr) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x) {
        out[i] = pw_sum_seq(a + off[i], len[i]);
        if (nonint) {   // integrality of the leaf's elements (their sums' exactness)
            bool bad = false;
            for (int64_t q = 0; q < len[i] && !bad; q++) bad = a[off[i] + q] != floor(a[off[i] + q]);
            if (bad) atomicOr(nonint, 1u);
        }
    }
}

__global__ void k_degree_bins(const int64_t *uptr, int64_t n, int64_t *flags, int32_t *maxdeg) {
    // flags: NBINS arrays of n+1 entries
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t d = uptr[r + 1] - uptr[r];
        int bin = -1;
        if (d > 0) {
            bin = 0;
            while (d > bin_hi(bin)) bin++;
        }
        for (int b = 0; b < NBINS; b++) flags[b * (n + 1) + r] = (b == bin);
        if (d > 0) atomicMax(maxdeg, (int32_t)(d > 0x7fffffff ? 0x7fffffff : d));
    }
}

__global__ void k_make_u32(const double *uu, int64_t ue, const double *s_out, const double *s_in,
                           int64_t n, uint32_t *u32, int32_t *bad, double2 *s2) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = t; e < ue; e += stride) {
        double x = uu[e];
        if (!(x >= 0.0 && x < 4294967296.0 && x == floor(x))) atomicOr(bad, 1);
        else u32[e] = (uint32_t)x;
    }
    for (int64_t r = t; r < n; r += stride) {
        if (!(s_out[r] + s_in[r] < 4294967296.0)) atomicOr(bad, 1);
        s2[r] = make_double2(s_out[r], s_in[r]);
    }
}

__global__ void k_scatter_bin(const int64_t *flag, const int64_t *pos, int64_t n, int64_t base,
                              int32_t *rows) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        if (flag[r]) rows[base + pos[r]] = (int32_t)r;
}

// ------------------------------------------------------------------- host side

// numpy pairwise sum of a device array, bit-identical to ndarray.sum(): the host walks the
// top of numpy's recursion down to segments of <= 32768 elements (each a node of the same
// recursion), one device thread sums each segment with the identical recursion, and the host
// recombines the partial sums in the recursion's order.
static void pw_segments(int64_t off, int64_t n, std::vector<int64_t> &offs,
                        std::vector<int64_t> &lens) {
    if (n <= 32768) {
        offs.push_back(off);
        lens.push_back(n);
        return;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    pw_segments(off, n2, offs, lens);
    pw_segments(off + n2, n - n2, offs, lens);
}
static double pw_combine(int64_t n, const double *vals, size_t &k) {
    if (n <= 32768) return vals[k++];
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    double l = pw_combine(n2, vals, k);
    double r = pw_combine(n - n2, vals, k);
    return l + r;
}

double device_pairwise_sum(slm_ctx *ctx, const double *d_a, int64_t n) {
    if (n == 0) return 0.0;
    std::vector<int64_t> offs, lens;
    pw_segments(0, n, offs, lens);
    int64_t k = (int64_t)offs.size();
    DBuf<int64_t> d_off, d_len;
    DBuf<double> d_out;
    d_off.resize(k);
    d_len.resize(k);
    d_out.resize(k);
    CUDA_TRY(cudaMemcpyAsync(d_off.p, offs.data(), k * 8, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(d_len.p, lens.data(), k * 8, cudaMemcpyHostToDevice, ctx->stream));
    k_pw_segments<<<grid_for(k, 128), 128, 0, ctx->stream>>>(d_a, d_off.p, d_len.p, k, d_out.p);
    std::vector<double> h(k);
    CUDA_TRY(cudaMemcpyAsync(h.data(), d_out.p, k * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    size_t idx = 0;
    return pw_combine(n, h.data(), idx);
}

void build_bins(slm_ctx *ctx, LevelGraph &G) {
    int64_t n = G.n;
    cudaStream_t s = ctx->stream;
    DBuf<int64_t> f, p;
    f.resize((n + 1) * NBINS);
    p.resize(n + 1);
    int32_t *d_max = ctx->i32d.resize(1);
    CUDA_TRY(cudaMemsetAsync(d_max, 0, 4, s));
    k_degree_bins<<<grid_for(n, 256), 256, 0, s>>>(G.uptr.p, n, f.p, d_max);
    int64_t tot[NBINS];
    G.bin_rows.resize(n > 0 ? n : 1);
    G.bin_off[0] = 0;
    for (int b = 0; b < NBINS; b++) {
        int64_t *fb = f.p + b * (n + 1);
        CUDA_TRY(cudaMemsetAsync(fb + n, 0, 8, s));
        dev_exclusive_sum<int64_t, int64_t>(ctx, fb, p.p, n + 1);
        CUDA_TRY(cudaMemcpyAsync(&tot[b], p.p + n, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        G.bin_off[b + 1] = G.bin_off[b] + tot[b];
        if (tot[b])
            k_scatter_bin<<<grid_for(n, 256), 256, 0, s>>>(fb, p.p, n, G.bin_off[b], G.bin_rows.p);
    }
    int32_t mx = 0;
    CUDA_TRY(cudaMemcpyAsync(&mx, d_max, 4, cudaMemcpyDeviceToHost, s));
    std::vector<int32_t> rows(G.bin_off[NBINS]);
    std::vector<int64_t> up(n + 1);
    if (!rows.empty())
        CUDA_TRY(cudaMemcpyAsync(rows.data(), G.bin_rows.p, rows.size() * 4,
                                 cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(up.data(), G.uptr.p, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    G.max_deg = mx;
    // bin 0 stably partitioned by degree: rows with d <= TINY_MAX first (the lane-per-row
    // kernel), then the rest; both parts keep ascending row ids (their union entries and row
    // metadata stay nearly sequential in memory)
    {
        const int64_t nb0 = G.bin_off[1] - G.bin_off[0];
        std::vector<int32_t> part(nb0);
        int64_t k0 = 0;
        for (int64_t k = 0; k < nb0; k++)
            if (up[rows[k] + 1] - up[rows[k]] <= TINY_MAX) part[k0++] = rows[k];
        G.bin0_tiny = k0;
        for (int64_t k = 0; k < nb0; k++)
            if (up[rows[k] + 1] - up[rows[k]] > TINY_MAX) part[k0++] = rows[k];
        std::copy(part.begin(), part.end(), rows.begin());
        if (nb0)
            CUDA_TRY(cudaMemcpyAsync(G.bin_rows.p, rows.data(), nb0 * 4, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
    for (int b = 0; b < NBINS; b++) {
        int64_t e = 0;
        for (int64_t k = G.bin_off[b]; k < G.bin_off[b + 1]; k++) e += up[rows[k] + 1] - up[rows[k]];
        G.bin_entries[b] = e;
    }
    // global hash scratch offsets for rows with d > MID_MAX (capacity next pow2 > d)
    const int64_t b0 = G.bin_off[4], nl = G.bin_off[NBINS] - b0;
    G.large_hash_total = 0;
    if (nl) {
        std::vector<int64_t> hoff(nl + 1);
        int64_t acc = 0;
        for (int64_t i = 0; i < nl; i++) {
            int64_t d = up[rows[b0 + i] + 1] - up[rows[b0 + i]];
            int64_t cap = 32;
            while (cap <= d) cap <<= 1;   // > d >= distinct communities of the row
            hoff[i] = acc;
            acc += cap;
        }
        hoff[nl] = acc;
        G.large_hash_total = acc;
        // hub rows (bin 5) for the integer sweep: processing order j = descending degree,
        // work items (j << 20 | segment) of HUB_SEG entries; row j's global table (pow2 > d
        // slots) and list are its own region of the hub arena
        const int64_t nb4 = G.bin_off[5] - G.bin_off[4];
        const int64_t nh = nl - nb4;
        std::vector<int64_t> hub(nh);
        for (int64_t j = 0; j < nh; j++) hub[j] = j;
        auto deg5 = [&](int64_t j) { return up[rows[b0 + nb4 + j] + 1] - up[rows[b0 + nb4 + j]]; };
        std::stable_sort(hub.begin(), hub.end(),
                         [&](int64_t x, int64_t y) { return deg5(x) > deg5(y); });
        std::vector<int64_t> segs, hoffr(nh), hsz(nh);
        int64_t cur = 0;
        for (int64_t j = 0; j < nh; j++) {
            const int64_t d = deg5(hub[j]);
            int64_t H = 64;
            while (H <= d) H <<= 1;
            hoffr[j] = cur;
            hsz[j] = H;
            cur += H;
            for (int64_t q = 0; q * HUB_SEG < d; q++) segs.push_back((j << 20) | q);
        }
        G.hub_rows_n = nh;
        G.hub_ring = cur;
        G.hub_nseg = (int64_t)segs.size();
        // the largest rows (a prefix in processing order) are spread over CTAs by segment;
        // the rest are processed one CTA per row
        G.hub_big_rows = 0;
        G.hub_big_items = 0;
        for (int64_t j = 0; j < nh && deg5(hub[j]) > HUB_BIG_DEG; j++) {
            G.hub_big_rows++;
            G.hub_big_items += (deg5(hub[j]) + HUB_SEG - 1) / HUB_SEG;
        }
        if (nh) {
            G.hub_seg.resize(segs.size());
            G.hub_row.resize(nh);
            G.hub_off.resize(nh);
            G.hub_size.resize(nh);
            CUDA_TRY(cudaMemcpyAsync(G.hub_seg.p, segs.data(), segs.size() * 8, cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaMemcpyAsync(G.hub_row.p, hub.data(), nh * 8, cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaMemcpyAsync(G.hub_off.p, hoffr.data(), nh * 8, cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaMemcpyAsync(G.hub_size.p, hsz.data(), nh * 8, cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaStreamSynchronize(s));
        }
        G.large_hoff.resize(nl + 1);
        CUDA_TRY(cudaMemcpyAsync(G.large_hoff.p, hoff.data(), (nl + 1) * 8,
                                 cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
}

// Long duplicate runs, all at once: run ends by binary search on the group ids, the numpy
// reduceat sum first + pairwise(rest) of every run from one batched leaf kernel (the host walks
// each run's pairwise recursion down to <= 32768-element leaves and recombines in its order),
// and one integrality check kernel.
__global__ void k_long_ends(const uint64_t *keys, int64_t ne, const int64_t *runs, int32_t nruns,
                            int64_t *ends) {
    for (int32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nruns; q += gridDim.x * blockDim.x) {
        const int64_t e = runs[2 * q];
        const uint64_t key = keys[e];
        int64_t lo = e, hi = ne;   // first index with a larger key (keys sorted)
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] <= key) lo = mid + 1;
            else hi = mid;
        }
        ends[q] = lo;
    }
}
__global__ void k_scatter_sums(const int64_t *runs, const double *sums, int32_t nruns, double *w) {
    for (int32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nruns; q += gridDim.x * blockDim.x)
        w[runs[2 * q + 1]] = sums[q];
}

static void merge_long_runs(slm_ctx *ctx, const double *vals, const uint64_t *keys, int64_t ne,
                            const int64_t *d_runs, int32_t nruns, double *out_w, uint32_t *bad) {
    cudaStream_t s = ctx->stream;
    CTX_SCRATCH(DBuf<int64_t>, ends);
    CTX_SCRATCH(DBuf<int64_t>, d_off);
    CTX_SCRATCH(DBuf<int64_t>, d_len);
    CTX_SCRATCH(DBuf<double>, leaf);
    CTX_SCRATCH(DBuf<double>, sums);
    ends.resize(nruns);
    k_long_ends<<<grid_for(nruns, 128), 128, 0, s>>>(keys, ne, d_runs, nruns, ends.p);
    std::vector<int64_t> hr(2 * nruns), he(nruns);
    CUDA_TRY(cudaMemcpyAsync(hr.data(), d_runs, nruns * 16, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(he.data(), ends.p, nruns * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<int64_t> offs, lens, first_leaf(nruns + 1), firsts(nruns);
    for (int32_t q = 0; q < nruns; q++) {
        first_leaf[q] = (int64_t)offs.size();
        offs.push_back(hr[2 * q]);   // leaf 0 of a run: its first element alone
        lens.push_back(1);
        pw_segments(hr[2 * q] + 1, he[q] - hr[2 * q] - 1, offs, lens);
    }
    first_leaf[nruns] = (int64_t)offs.size();
    const int64_t nl = (int64_t)offs.size();
    d_off.resize(nl);
    d_len.resize(nl);
    leaf.resize(nl);
    CUDA_TRY(cudaMemcpyAsync(d_off.p, offs.data(), nl * 8, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(d_len.p, lens.data(), nl * 8, cudaMemcpyHostToDevice, s));
    // (the leaves cover every element of the runs: their integrality is checked there, by
    // the ~32K-element leaves in parallel, not one CTA per run)
    k_pw_segments<<<grid_for(nl, 128), 128, 0, s>>>(vals, d_off.p, d_len.p, nl, leaf.p, bad);
    std::vector<double> hl(nl), hs(nruns);
    CUDA_TRY(cudaMemcpyAsync(hl.data(), leaf.p, nl * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int32_t q = 0; q < nruns; q++) {
        size_t k = (size_t)first_leaf[q] + 1;
        const double rest = pw_combine(he[q] - hr[2 * q] - 1, hl.data(), k);
        hs[q] = hl[first_leaf[q]] + rest;
    }
    sums.resize(nruns);
    CUDA_TRY(cudaMemcpyAsync(sums.p, hs.data(), nruns * 8, cudaMemcpyHostToDevice, s));
    k_scatter_sums<<<grid_for(nruns, 128), 128, 0, s>>>(d_runs, sums.p, nruns, out_w);
    CUDA_TRY(cudaStreamSynchronize(s));
}

void build_level_from_keys(slm_ctx *ctx, LevelGraph &G, int64_t n, DBuf<uint64_t> &keys,
                           DBuf<double> &vals, int64_t ne_in) {
    cudaStream_t s = ctx->stream;
    const bool aprof = getenv("SLM_PROFILE_AGG") != nullptr;
    double at0 = now_ms();
    auto amark = [&](const char *what) {
        if (!aprof) return;
        CUDA_TRY(cudaStreamSynchronize(s));
        const double t = now_ms();
        fprintf(stderr, "[level build n=%lld ne=%lld] %s %.2f ms\n", (long long)n, (long long)ne_in,
                what, t - at0);
        at0 = t;
    };
    amark("start");
    const int b = bits_for(n);
    SLM_REQUIRE(n < (int64_t(1) << 31), SLM_EUNSUP, "more than 2^31-1 nodes");
    G.n = n;
    // 1. stable sort by (src, dst)
    if (ne_in > 0) sort_pairs_u64_f64(ctx, keys, vals, ne_in, 2 * b);
    amark("sort");
    // 2. run heads + group ids
    CTX_SCRATCH(DBuf<int64_t>, head);   // grow-only scratch kept across builds
    CTX_SCRATCH(DBuf<int64_t>, gid);
    head.resize(ne_in + 1);
    gid.resize(ne_in + 1);
    int64_t ng = 0;
    uint32_t *d_int_bad = (uint32_t *)ctx->i32d.resize(2);
    CUDA_TRY(cudaMemsetAsync(d_int_bad, 0, 8, s));
    if (ne_in > 0) {
        k_run_heads<<<grid_for(ne_in, 256), 256, 0, s>>>(keys.p, ne_in, head.p);
        CUDA_TRY(cudaMemsetAsync(head.p + ne_in, 0, 8, s));
        dev_exclusive_sum<int64_t, int64_t>(ctx, head.p, gid.p, ne_in + 1);
        CUDA_TRY(cudaMemcpyAsync(&ng, gid.p + ne_in, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
    SLM_REQUIRE(ng < (int64_t(1) << 31), SLM_EUNSUP, "more than 2^31-1 merged edges");
    G.ne = ng;
    CTX_SCRATCH(DBuf<int32_t>, src_of);   // grow-only scratch kept across builds
    src_of.resize(ng);
    G.csr_dst.resize(ng);
    G.csr_w.resize(ng);
    G.csr_ptr.resize(n + 1);
    if (ne_in > 0) {
        CTX_SCRATCH(DBuf<int64_t>, lr);
        lr.resize(2 * MAX_LONG + 2);
        int32_t *d_nlong = (int32_t *)(lr.p + 2 * MAX_LONG);
        CUDA_TRY(cudaMemsetAsync(d_nlong, 0, 4, s));
        k_merge_runs<<<grid_for(ne_in, 256), 256, 0, s>>>(keys.p, vals.p, gid.p, ne_in, b,
                                                          src_of.p, G.csr_dst.p, G.csr_w.p,
                                                          d_int_bad, lr.p, d_nlong);
        int32_t nlong = 0;
        CUDA_TRY(cudaMemcpyAsync(&nlong, d_nlong, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        SLM_REQUIRE(nlong <= MAX_LONG, SLM_EUNSUP, "too many long duplicate runs");
        if (nlong) merge_long_runs(ctx, vals.p, keys.p, ne_in, lr.p, nlong, G.csr_w.p, d_int_bad);
    }
    k_lower_bound_ptr<<<grid_for(n + 1, 256), 256, 0, s>>>(src_of.p, ng, n, G.csr_ptr.p);
    amark("merge runs");
    amark("release");
    // 3. stable transpose (in-CSR, graph.py:111-115): sort entry ids by dst
    DBuf<int64_t> in_ptr;
    DBuf<int32_t> in_src;
    DBuf<double> in_w;
    in_ptr.resize(n + 1);
    in_src.resize(ng);
    in_w.resize(ng);
    {
        CTX_SCRATCH(DBuf<int32_t>, perm_in);   // grow-only scratch kept across builds
        CTX_SCRATCH(DBuf<int32_t>, perm_out);
        CTX_SCRATCH(DBuf<int32_t>, kout);
        perm_in.resize(ng);
        perm_out.resize(ng);
        kout.resize(ng);
        amark("transpose alloc");
        k_iota_i32<<<grid_for(ng, 256), 256, 0, s>>>(perm_in.p, ng);
        if (ng > 0)
            sort_pairs_u32_i32(ctx, (uint32_t *)G.csr_dst.p, (uint32_t *)kout.p, perm_in.p,
                               perm_out.p, ng, b);
        amark("transpose sort");
        k_gather_transpose<<<grid_for(ng, 256), 256, 0, s>>>(perm_out.p, src_of.p, G.csr_w.p, ng,
                                                             in_src.p, in_w.p);
        k_lower_bound_ptr<<<grid_for(n + 1, 256), 256, 0, s>>>(kout.p, ng, n, in_ptr.p);
    }
    amark("transpose");
    // 4. symmetric?
    int32_t *d_asym = ctx->i32c.resize(1);
    CUDA_TRY(cudaMemsetAsync(d_asym, 0, 4, s));
    k_sym_check<<<grid_for(ng + n, 256), 256, 0, s>>>(G.csr_ptr.p, G.csr_dst.p, G.csr_w.p,
                                                      in_ptr.p, in_src.p, in_w.p, n, ng, d_asym);
    int32_t asym = 0;
    uint32_t intbad[2] = {0, 0};
    CUDA_TRY(cudaMemcpyAsync(&asym, d_asym, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(intbad, d_int_bad, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    G.sym = (asym == 0);
    amark("sym check");
    // 5. union
    if (G.sym) {
        CTX_SCRATCH(DBuf<int64_t>, keep);   // grow-only scratch kept across builds
        CTX_SCRATCH(DBuf<int64_t>, pos);
        keep.resize(ng + 1);
        pos.resize(ng + 1);
        CUDA_TRY(cudaMemsetAsync(keep.p, 0, (ng + 1) * 8, s));
        k_keep_nonself<<<grid_for(n * 32, 256), 256, 0, s>>>(G.csr_ptr.p, G.csr_dst.p, n, keep.p);
        dev_exclusive_sum<int64_t, int64_t>(ctx, keep.p, pos.p, ng + 1);
        int64_t ue = 0;
        CUDA_TRY(cudaMemcpyAsync(&ue, pos.p + ng, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        G.ue = ue;
        G.uptr.resize(n + 1);
        G.unbr.resize(ue);
        G.uu.resize(ue);
        k_fill_union_sym<<<grid_for(n * 32, 256), 256, 0, s>>>(G.csr_ptr.p, G.csr_dst.p,
                                                              G.csr_w.p, pos.p, n, ng, ue,
                                                              G.uptr.p, G.unbr.p, G.uu.p);
    } else {
        CTX_SCRATCH(DBuf<int64_t>, cnt);   // grow-only scratch kept across builds
        cnt.resize(n + 1);
        CUDA_TRY(cudaMemsetAsync(cnt.p + n, 0, 8, s));
        k_union_merge<<<grid_for(n, 128), 128, 0, s>>>(G.csr_ptr.p, G.csr_dst.p, G.csr_w.p,
                                                       in_ptr.p, in_src.p, in_w.p, n, 0, cnt.p,
                                                       nullptr, nullptr);
        G.uptr.resize(n + 1);
        dev_exclusive_sum<int64_t, int64_t>(ctx, cnt.p, G.uptr.p, n + 1);
        int64_t ue = 0;
        CUDA_TRY(cudaMemcpyAsync(&ue, G.uptr.p + n, 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        G.ue = ue;
        G.unbr.resize(ue);
        G.uu.resize(ue);
        k_union_merge<<<grid_for(n, 128), 128, 0, s>>>(G.csr_ptr.p, G.csr_dst.p, G.csr_w.p,
                                                       in_ptr.p, in_src.p, in_w.p, n, 1,
                                                       G.uptr.p, G.unbr.p, G.uu.p);
    }
    amark("union");
    // 6. strengths
    G.s_out.resize(n);
    G.s_in.resize(n);
    k_row_seq_sum<<<grid_for(n, 128), 128, 0, s>>>(G.csr_ptr.p, G.csr_w.p, n, G.s_out.p);
    if (G.sym)
        CUDA_TRY(cudaMemcpyAsync(G.s_in.p, G.s_out.p, n * 8, cudaMemcpyDeviceToDevice, s));
    else
        k_row_seq_sum<<<grid_for(n, 128), 128, 0, s>>>(in_ptr.p, in_w.p, n, G.s_in.p);
    G.m_w = device_pairwise_sum(ctx, G.csr_w.p, ng);
    G.integral = (intbad[0] == 0) && (G.m_w < 9007199254740992.0);
    amark("strengths");
    build_bins(ctx, G);
    amark("bins");
    // compact integer weights for the plan sweep's fast path, interleaved strengths
    G.s2.resize(n);
    G.u32_ok = false;
    if (G.integral) {
        G.uu32.resize(G.ue);
        int32_t *d_bad = ctx->i32c.resize(1);
        CUDA_TRY(cudaMemsetAsync(d_bad, 0, 4, s));
        k_make_u32<<<grid_for(std::max<int64_t>(G.ue, n), 256), 256, 0, s>>>(
            G.uu.p, G.ue, G.s_out.p, G.s_in.p, n, G.uu32.p, d_bad, G.s2.p);
        int32_t hb = 0;
        CUDA_TRY(cudaMemcpyAsync(&hb, d_bad, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        G.u32_ok = (hb == 0);
        if (!G.u32_ok) G.uu32.release();
    } else {
        int32_t *d_bad = ctx->i32c.resize(1);
        k_make_u32<<<grid_for(n, 256), 256, 0, s>>>(G.uu.p, 0, G.s_out.p, G.s_in.p, n, nullptr,
                                                      d_bad, G.s2.p);
    }
    CUDA_TRY(cudaStreamSynchronize(s));
}

void build_level_from_edges(slm_ctx *ctx, LevelGraph &G, int64_t n, const int32_t *d_src,
                            const int32_t *d_dst, const double *d_w, int64_t ne_in) {
    cudaStream_t s = ctx->stream;
    int32_t *d_bad = ctx->i32c.resize(1);
    CUDA_TRY(cudaMemsetAsync(d_bad, 0, 4, s));
    if (ne_in > 0)
        k_validate<<<grid_for(ne_in, 256), 256, 0, s>>>(d_src, d_dst, d_w, ne_in, n, d_bad);
    int32_t bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    SLM_REQUIRE(!(bad & 1), SLM_EINVAL, "edge endpoint out of range");
    SLM_REQUIRE(!(bad & 2), SLM_EINVAL, "edge weights must be finite and positive");
    DBuf<uint64_t> keys;
    DBuf<double> vals;
    keys.resize(ne_in);
    vals.resize(ne_in);
    if (ne_in > 0)
        k_make_keys<<<grid_for(ne_in, 256), 256, 0, s>>>(d_src, d_dst, d_w, ne_in, bits_for(n),
                                                         keys.p, vals.p);
    build_level_from_keys(ctx, G, n, keys, vals, ne_in);
}

// ------------------------------------------------- degree-ordered view of the union

__global__ void k_view_keys(const int64_t *uptr, int64_t n, uint32_t *key, int32_t *idx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        key[i] = ~(uint32_t)(uptr[i + 1] - uptr[i]);   // ascending key = descending degree
        idx[i] = (int32_t)i;
    }
}

__global__ void k_view_rows(const int64_t *uptr, const int32_t *order, int64_t n, int64_t *vdeg,
                            int32_t *newid) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = order[k];
        vdeg[k] = uptr[v + 1] - uptr[v];
        newid[v] = (int32_t)k;
    }
}

// one warp per view row: entries copied in order, neighbours renumbered
__global__ void k_view_entries(const int64_t *uptr, const int32_t *unbr, const uint32_t *u32,
                               const int32_t *order, const int32_t *newid, int64_t n,
                               const int64_t *vptr, int32_t *vnbr, uint32_t *vu32) {
    const int lane = threadIdx.x & 31;
    for (int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; k < n;
         k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t v = order[k];
        const int64_t s0 = uptr[v], d = uptr[v + 1] - s0, t0 = vptr[k];
        for (int64_t t = lane; t < d; t += 32) {
            vnbr[t0 + t] = newid[unbr[s0 + t]];
            vu32[t0 + t] = u32[s0 + t];
        }
    }
}

// Sorted form of the view's rows (neighbours ascending in VIEW numbering), by transposition:
// the union's pattern and u = w_out + w_in are symmetric, so a stable sort of the view's
// row-major entries (k, j, u) by the destination j groups them by j with k ascending --
// which is row j of the view with its neighbours in ascending order.  Key = j, payload =
// (k, u); row offsets are unchanged (deg is symmetric too).  Hub neighbours (the low view
// ids) then sit at the front of every row and the label gathers of consecutive lanes share
// 128-byte lines.
__global__ void k_view_entries_kv(const int64_t *uptr, const int32_t *unbr, const uint32_t *u32,
                                  const int32_t *order, const int32_t *newid, int64_t n,
                                  const int64_t *vptr, uint32_t *key, uint64_t *val) {
    const int lane = threadIdx.x & 31;
    for (int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; k < n;
         k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t v = order[k];
        const int64_t s0 = uptr[v], d = uptr[v + 1] - s0, t0 = vptr[k];
        for (int64_t t = lane; t < d; t += 32) {
            key[t0 + t] = (uint32_t)newid[unbr[s0 + t]];
            val[t0 + t] = ((uint64_t)k << 32) | u32[s0 + t];
        }
    }
}
__global__ void k_view_split(const uint64_t *val, int64_t ue, int32_t *vnbr, uint32_t *vu32) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ue;
         e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t v = val[e];
        vnbr[e] = (int32_t)(v >> 32);
        vu32[e] = (uint32_t)v;
    }
}

template <class T>
__global__ void k_view_gather(const T *src, const int32_t *order, int64_t n, T *dst) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = src[order[k]];
}

// Bins of the view without flags or host passes: the view's degrees are non-increasing, so
// every degree bin (and bin 0's d <= TINY_MAX tail) is a contiguous range of view rows.
// bound[b] (b = 0..NBINS-1) = first row whose bin is below b (n if none); bound[NBINS] =
// first row of degree <= TINY_MAX.
__device__ __forceinline__ int view_bin(int64_t d) {
    if (d <= 0) return -1;
    int b = 0;
    while (d > bin_hi(b)) b++;
    return b;
}
__global__ void k_view_bounds(const int64_t *vptr, int64_t n, int64_t *bound) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = vptr[k + 1] - vptr[k];
        const int64_t dp = k ? vptr[k] - vptr[k - 1] : INT64_MAX;
        const int bk = view_bin(d), bp = k ? view_bin(dp) : NBINS;
        for (int b = bk + 1; b <= bp && b < NBINS; b++) bound[b] = k;
        if (d <= TINY_MAX && dp > TINY_MAX) bound[NBINS] = k;
        if (d <= HALF_MAX && dp > HALF_MAX) bound[NBINS + 1] = k;
    }
}
// rows[off + i] = start + i over up to 8 segments {off, start, len}
__global__ void k_view_fill_rows(const int64_t *seg, int nseg, int32_t *rows) {
    for (int q = 0; q < nseg; q++) {
        const int64_t off = seg[3 * q], st = seg[3 * q + 1], len = seg[3 * q + 2];
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
             i += (int64_t)gridDim.x * blockDim.x)
            rows[off + i] = (int32_t)(st + i);
    }
}

static void build_bins_view(slm_ctx *ctx, LevelGraph &V) {
    const int64_t n = V.n;
    cudaStream_t s = ctx->stream;
    int64_t *d_b = ctx->view_bound.resize(NBINS + 2 + 3 * 8);
    std::vector<int64_t> hb(NBINS + 2, n);
    CUDA_TRY(cudaMemcpyAsync(d_b, hb.data(), (NBINS + 2) * 8, cudaMemcpyHostToDevice, s));
    if (n) k_view_bounds<<<grid_for(n, 256), 256, 0, s>>>(V.uptr.p, n, d_b);
    CUDA_TRY(cudaMemcpyAsync(hb.data(), d_b, (NBINS + 2) * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    // bin b = view rows [lo(b), hi(b)): hi(b) = bound[b], lo(b) = bound[b + 1] (lo(5) = 0)
    auto lo = [&](int b) { return b == NBINS - 1 ? (int64_t)0 : hb[b + 1]; };
    auto hi = [&](int b) { return hb[b]; };
    // uptr at the boundaries
    std::vector<int64_t> cut;
    for (int b = 0; b < NBINS; b++) {
        cut.push_back(lo(b));
        cut.push_back(hi(b));
    }
    std::vector<int64_t> upc(cut.size());
    for (size_t q = 0; q < cut.size(); q++)
        CUDA_TRY(cudaMemcpyAsync(&upc[q], V.uptr.p + cut[q], 8, cudaMemcpyDeviceToHost, s));
    const int64_t t0 = std::max(lo(0), std::min(hi(0), hb[NBINS]));   // first tiny row of bin 0
    std::vector<int64_t> seg;
    int64_t off = 0;
    V.bin_rows.resize(n > 0 ? n : 1);
    for (int b = 0; b < NBINS; b++) {
        V.bin_off[b] = off;
        if (b == 0) {
            seg.insert(seg.end(), {off, t0, hi(0) - t0});   // d <= TINY_MAX first
            seg.insert(seg.end(), {off + hi(0) - t0, lo(0), t0 - lo(0)});
            V.bin0_tiny = hi(0) - t0;
        } else {
            seg.insert(seg.end(), {off, lo(b), hi(b) - lo(b)});
        }
        off += hi(b) - lo(b);
    }
    V.bin_off[NBINS] = off;
    // bin 1's rows of d <= HALF_MAX: the tail of its (descending-degree) segment
    V.bin1_half = hi(1) - std::max(lo(1), std::min(hi(1), hb[NBINS + 1]));
    CUDA_TRY(cudaMemcpyAsync(d_b + NBINS + 2, seg.data(), seg.size() * 8, cudaMemcpyHostToDevice, s));
    if (off) k_view_fill_rows<<<grid_for(off, 256), 256, 0, s>>>(d_b + NBINS + 2, (int)seg.size() / 3,
                                                                 V.bin_rows.p);
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int b = 0; b < NBINS; b++) V.bin_entries[b] = upc[2 * b + 1] - upc[2 * b];
    V.max_deg = 0;
    if (n) {
        int64_t u01[2];
        CUDA_TRY(cudaMemcpy(u01, V.uptr.p, 16, cudaMemcpyDeviceToHost));
        V.max_deg = (int32_t)std::min<int64_t>(u01[1] - u01[0], 0x7fffffff);
    }
    V.large_hash_total = 0;   // the generic fp64 path never runs on a view
    // hub rows (bin 5) = view rows [0, nh), already in descending degree: j = row
    const int64_t nh = hi(NBINS - 1) - lo(NBINS - 1);
    V.hub_rows_n = nh;
    V.hub_nseg = 0;
    V.hub_ring = 0;
    V.hub_big_rows = 0;
    V.hub_big_items = 0;
    if (nh) {
        std::vector<int64_t> up(nh + 1);
        CUDA_TRY(cudaMemcpy(up.data(), V.uptr.p, (nh + 1) * 8, cudaMemcpyDeviceToHost));
        std::vector<int64_t> hub(nh), segs, hoffr(nh), hsz(nh);
        int64_t cur = 0;
        for (int64_t j = 0; j < nh; j++) {
            hub[j] = j;
            const int64_t d = up[j + 1] - up[j];
            int64_t H = 64;
            while (H <= d) H <<= 1;
            hoffr[j] = cur;
            hsz[j] = H;
            cur += H;
            for (int64_t q = 0; q * HUB_SEG < d; q++) segs.push_back((j << 20) | q);
            if (d > HUB_BIG_DEG && V.hub_big_rows == j) {
                V.hub_big_rows++;
                V.hub_big_items += (d + HUB_SEG - 1) / HUB_SEG;
            }
        }
        V.hub_ring = cur;
        V.hub_nseg = (int64_t)segs.size();
        V.hub_seg.resize(segs.size());
        V.hub_row.resize(nh);
        V.hub_off.resize(nh);
        V.hub_size.resize(nh);
        CUDA_TRY(cudaMemcpyAsync(V.hub_seg.p, segs.data(), segs.size() * 8, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(V.hub_row.p, hub.data(), nh * 8, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(V.hub_off.p, hoffr.data(), nh * 8, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(V.hub_size.p, hsz.data(), nh * 8, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
}

SweepView &ensure_sweep_view(slm_ctx *ctx, const LevelGraph &G) {
    if (G.view) return *G.view;
    cudaStream_t s = ctx->stream;
    static const bool verbose = getenv("SLM_VIEW_VERBOSE") != nullptr;
    const double t_begin = now_ms();
    double tv = t_begin;
    auto vmark = [&](const char *what) {
        if (!verbose) return;
        cudaStreamSynchronize(s);
        const double t = now_ms();
        fprintf(stderr, "[view] %s %.1f ms\n", what, t - tv);
        tv = t;
    };
    auto W = std::make_shared<SweepView>();
    LevelGraph &V = W->V;
    const int64_t n = G.n, ue = G.ue;
    V.n = n;
    V.ne = 0;
    V.ue = ue;
    V.sym = G.sym;
    V.integral = G.integral;
    V.u32_ok = G.u32_ok;
    V.m_w = G.m_w;
    W->order.resize(n);
    W->vlabel.resize(n);
    W->vcstar.resize(n);
    {
        DBuf<uint32_t> &k0 = ctx->view_k0, &k1 = ctx->view_k1;
        DBuf<int32_t> &i0 = ctx->view_i0, &nid = ctx->view_nid;
        k0.resize(n);
        k1.resize(n);
        i0.resize(n);
        nid.resize(n);
        k_view_keys<<<grid_for(n, 256), 256, 0, s>>>(G.uptr.p, n, k0.p, i0.p);
        vmark("alloc+keys");
        sort_pairs_u32_i32(ctx, k0.p, k1.p, i0.p, W->order.p, n, 32);   // stable (LSD)
        vmark("sort");
        DBuf<int64_t> &vdeg = ctx->view_deg;
        vdeg.resize(n + 1);
        CUDA_TRY(cudaMemsetAsync(vdeg.p + n, 0, 8, s));
        k_view_rows<<<grid_for(n, 256), 256, 0, s>>>(G.uptr.p, W->order.p, n, vdeg.p, nid.p);
        V.uptr.resize(n + 1);
        dev_exclusive_sum<int64_t, int64_t>(ctx, vdeg.p, V.uptr.p, n + 1);
        V.unbr.resize(ue);
        V.uu32.resize(ue);
        static const bool sorted_rows =
            !(getenv("SLM_VIEW_SORTED") && atoi(getenv("SLM_VIEW_SORTED")) == 0);
        if (sorted_rows && ue > 0) {
            DBuf<uint32_t> kA, kB;
            DBuf<uint64_t> vA, vB;
            kA.resize(ue);
            kB.resize(ue);
            vA.resize(ue);
            vB.resize(ue);
            k_view_entries_kv<<<grid_for(n * 32, 256), 256, 0, s>>>(
                G.uptr.p, G.unbr.p, G.uu32.p, W->order.p, nid.p, n, V.uptr.p, kA.p, vA.p);
            vmark("entries (key, payload)");
            const bool inB = sort_pairs_u32_u64(ctx, kA.p, kB.p, vA.p, vB.p, ue, bits_for(n));
            vmark("transpose sort");
            k_view_split<<<grid_for(ue, 256), 256, 0, s>>>(inB ? vB.p : vA.p, ue, V.unbr.p,
                                                            V.uu32.p);
            CUDA_TRY(cudaStreamSynchronize(s));   // the local buffers go back to the arena
            vmark("split");
        } else {
            k_view_entries<<<grid_for(n * 32, 256), 256, 0, s>>>(G.uptr.p, G.unbr.p, G.uu32.p,
                                                                   W->order.p, nid.p, n, V.uptr.p,
                                                                   V.unbr.p, V.uu32.p);
            vmark("entries");
        }
    }
    V.s_out.resize(n);
    k_view_gather<double><<<grid_for(n, 256), 256, 0, s>>>(G.s_out.p, W->order.p, n, V.s_out.p);
    if (!G.sym) {
        V.s2.resize(n);
        k_view_gather<double2><<<grid_for(n, 256), 256, 0, s>>>(G.s2.p, W->order.p, n, V.s2.p);
    }
    CUDA_TRY(cudaGetLastError());
    vmark("strengths");
    build_bins_view(ctx, V);   // (ends with a stream synchronisation)
    vmark("bins");
    ctx->view_build_ms += now_ms() - t_begin;
    G.view = W;
    return *W;
}

// a kernel of this translation unit (module preloading, slm_capi.cu preload_modules)
const void *slm_anchor_build() { return (const void *)k_validate; }
