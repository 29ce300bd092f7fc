// slm_lgains.cu -- local gains (quality.py:170-183) and the POSITIVE trigger (bad
// communities, detector.py:342-345), integer fast path.
//
//   w_own[i] = sum of u_e over the entries of row i whose neighbour has label[i]
//   lg[i]    = (w_own / m) - ((s_out (S_in[c] - s_in) + s_in (S_out[c] - s_out)) / (m m))
//
// With integer weights (LevelGraph::u32_ok) w_own is an exact uint32 sum, so any summation
// order reproduces the reference's fp64 value; the final expression keeps its operand order.
// Rows are processed by degree bin (slm_internal.cuh): d <= 32 packed into warps (segmented
// shuffle sums), up to 4096 one warp per row, larger one CTA per row; rows without entries
// (w_own = 0) by a separate pass.
#include "slm_internal.cuh"

struct LGArgs {
    const int64_t *uptr;
    const int32_t *unbr;
    const uint32_t *u32;
    const int32_t *label;
    const double *S_out, *S_in, *s_out, *s_in;
    double m;
    double *lg;
    uint8_t *bad;
    const int32_t *order;   // rows of a sweep view: view row -> node (nullptr: rows are nodes)
};

__device__ __forceinline__ void lg_finish(const LGArgs &A, int32_t r, int32_t L, uint32_t own) {
    const double so = A.s_out[r], si = A.s_in[r];
    double g = (double)own / A.m - (so * (A.S_in[L] - si) + si * (A.S_out[L] - so)) / (A.m * A.m);
    if (A.m == 0.0) g = 0.0;
    if (A.lg) A.lg[A.order ? A.order[r] : r] = g;
    if (g < 0.0) A.bad[L] = 1;
}

// bin 0: rows packed into warps (lane = entry), segmented inclusive sums per row
__global__ void __launch_bounds__(256) k_lg_small(LGArgs A, const int32_t *rows, int64_t nrows) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t per = 64;   // rows per warp task
    for (int64_t base = w * per; base < nrows; base += nw * per) {
        const int64_t rend = min(base + per, nrows);
        int64_t rcur = base;
        while (rcur < rend) {
            const int64_t j = rcur + lane;
            int32_t r = 0, L = 0;
            int64_t e0 = 0;
            int deg = 0;
            if (j < rend) {
                r = rows[j];
                e0 = A.uptr[r];
                deg = (int)(A.uptr[r + 1] - e0);
                L = A.label[r];
            }
            int inc = deg;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, inc, off);
                if (lane >= off) inc += v;
            }
            const unsigned fit = __ballot_sync(0xffffffffu, j < rend && inc <= 32);
            const int k = __popc(fit);
            const int start = inc - deg;
            const int total = __shfl_sync(0xffffffffu, inc, k - 1);
            int s = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int cand = s + step;
                const int st = __shfl_sync(0xffffffffu, start, cand & 31);
                if (cand < k && st <= lane) s = cand;
            }
            const bool valid = lane < total;
            const int64_t re0 = __shfl_sync(0xffffffffu, e0, s);
            const int rst = __shfl_sync(0xffffffffu, start, s);
            const int32_t Lr = __shfl_sync(0xffffffffu, L, s);
            uint32_t v = 0;
            if (valid) {
                const int64_t e = re0 + (lane - rst);
                if (A.label[__ldcs(A.unbr + e)] == Lr) v = __ldcs(A.u32 + e);
            }
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, v, off);
                const int os = __shfl_up_sync(0xffffffffu, s, off);
                if (lane >= off && os == s) v += o;
            }
            const int nxt = __shfl_down_sync(0xffffffffu, s, 1);
            const bool last = valid && (lane == total - 1 || nxt != s);
            const int32_t rr = __shfl_sync(0xffffffffu, r, s);
            if (last) lg_finish(A, rr, Lr, v);
            rcur += k;
        }
    }
}

// bins 1-3: one warp per row
__global__ void __launch_bounds__(256) k_lg_warp(LGArgs A, const int32_t *rows, int64_t nrows) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i < nrows; i += nw) {
        const int32_t r = rows[i];
        const int64_t e0 = A.uptr[r];
        const uint32_t d = (uint32_t)(A.uptr[r + 1] - e0);
        const int32_t L = A.label[r];
        const int32_t *nb = A.unbr + e0;
        const uint32_t *ub = A.u32 + e0;
        uint32_t own = 0;
        constexpr int U = 4;
        for (uint32_t cb = lane; cb < d; cb += 32 * U) {
            int32_t z[U];
            uint32_t u[U];
#pragma unroll
            for (int q = 0; q < U; q++) {
                const uint32_t idx = cb + q * 32;
                z[q] = idx < d ? __ldcs(nb + idx) : -1;
                u[q] = idx < d ? __ldcs(ub + idx) : 0u;
            }
#pragma unroll
            for (int q = 0; q < U; q++)
                if (z[q] >= 0 && A.label[z[q]] == L) own += u[q];
        }
        own = __reduce_add_sync(0xffffffffu, own);
        if (lane == 0) lg_finish(A, r, L, own);
    }
}

// bins 4-5: one CTA per row
__global__ void __launch_bounds__(256) k_lg_cta(LGArgs A, const int32_t *rows, int64_t nrows) {
    __shared__ uint32_t part[8];
    for (int64_t i = blockIdx.x; i < nrows; i += gridDim.x) {
        const int32_t r = rows[i];
        const int64_t e0 = A.uptr[r];
        const int64_t d = A.uptr[r + 1] - e0;
        const int32_t L = A.label[r];
        uint32_t own = 0;
        constexpr int U = 4;
        for (int64_t cb = threadIdx.x; cb < d; cb += 256 * U) {
            int32_t z[U];
            uint32_t u[U];
#pragma unroll
            for (int q = 0; q < U; q++) {
                const int64_t idx = cb + q * 256;
                z[q] = idx < d ? __ldcs(A.unbr + e0 + idx) : -1;
                u[q] = idx < d ? __ldcs(A.u32 + e0 + idx) : 0u;
            }
#pragma unroll
            for (int q = 0; q < U; q++)
                if (z[q] >= 0 && A.label[z[q]] == L) own += u[q];
        }
        own = __reduce_add_sync(0xffffffffu, own);
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = own;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int k = 0; k < 8; k++) t += part[k];
            lg_finish(A, r, L, t);
        }
        __syncthreads();
    }
}

// rows without union entries: w_own = 0
__global__ void k_lg_empty(LGArgs A, int64_t n) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        if (A.uptr[r + 1] == A.uptr[r]) lg_finish(A, (int32_t)r, A.label[r], 0u);
}

// Symmetric graphs run over the level's degree-ordered sweep view (slm_build.cu), whose
// neighbour-label gathers stay in L2: labels are gathered into view order first and lg is
// written back at the node (w_own is an exact integer sum, so the order is immaterial).
void run_local_gains_u32(slm_ctx *ctx, const LevelGraph &G_, Forest &F, double m, double *d_lg,
                         uint8_t *d_bad) {
    cudaStream_t s = ctx->stream;
    static const bool no_view = getenv("SLM_VIEW") && atoi(getenv("SLM_VIEW")) == 0;
    const bool use_view = G_.sym && !no_view;
    const LevelGraph *gp = &G_;
    const int32_t *label = F.comm.p, *order = nullptr;
    if (use_view) {
        SweepView &W = ensure_sweep_view(ctx, G_);
        view_gather_labels(ctx, W, F.comm.p);
        gp = &W.V;
        label = W.vlabel.p;
        order = W.order.p;
    }
    const LevelGraph &G = *gp;
    LGArgs A;
    A.uptr = G.uptr.p;
    A.unbr = G.unbr.p;
    A.u32 = G.uu32.p;
    A.label = label;
    A.S_out = F.S_out.p;
    A.S_in = F.S_in.p;
    A.s_out = G.s_out.p;
    A.s_in = use_view ? G.s_out.p : G.s_in.p;   // symmetric: s_in == s_out bitwise
    A.m = m;
    A.lg = d_lg;
    A.bad = d_bad;
    A.order = order;
    auto nb = [&](int b0, int b1) { return G.bin_off[b1] - G.bin_off[b0]; };
    const int32_t *rows = G.bin_rows.p;
    if (nb(0, 1)) {
        const int64_t tasks = (nb(0, 1) + 63) / 64;
        k_lg_small<<<grid_for(tasks * 32, 256), 256, 0, s>>>(A, rows + G.bin_off[0], nb(0, 1));
    }
    if (nb(1, 4))
        k_lg_warp<<<grid_for(nb(1, 4) * 32, 256), 256, 0, s>>>(A, rows + G.bin_off[1], nb(1, 4));
    if (nb(4, NBINS))
        k_lg_cta<<<(unsigned)std::min<int64_t>(nb(4, NBINS), SMS() * 8), 256, 0, s>>>(
            A, rows + G.bin_off[4], nb(4, NBINS));
    if (G.n) k_lg_empty<<<grid_for(G.n, 256), 256, 0, s>>>(A, G.n);
    CUDA_TRY(cudaGetLastError());
}

// a kernel of this translation unit (module preloading, slm_capi.cu preload_modules)
const void *slm_anchor_lgains() { return (const void *)k_lg_small; }

// local gains from the own-community sums the integer sweep left (ctx->wown, kept exact across
// commits): one pass over the nodes instead of one over the union
__global__ void k_lg_wown(LGArgs A, const uint32_t *wown, int64_t n) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        lg_finish(A, (int32_t)r, A.label[r], wown[r]);
}
void run_local_gains_wown(slm_ctx *ctx, const LevelGraph &G, Forest &F, double m,
                          const uint32_t *wown, double *d_lg, uint8_t *d_bad) {
    LGArgs A;
    A.uptr = G.uptr.p;
    A.unbr = G.unbr.p;
    A.u32 = G.uu32.p;
    A.label = F.comm.p;
    A.S_out = F.S_out.p;
    A.S_in = F.S_in.p;
    A.s_out = G.s_out.p;
    A.s_in = G.s_in.p;
    A.m = m;
    A.lg = d_lg;
    A.bad = d_bad;
    A.order = nullptr;
    if (G.n) k_lg_wown<<<grid_for(G.n, 256), 256, 0, ctx->stream>>>(A, wown, G.n);
    CUDA_TRY(cudaGetLastError());
}
