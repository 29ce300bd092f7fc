// slm_forest.cu -- assignment forest structure on the device.
//
//   extract_components (forest.py:43-67)   -> run_components: cycle detection, root
//       pointers, min-cycle-id key, canonical dense labels by smallest member
//       (canonicalize_labels, graph.py:283-291).
//   community_members (forest.py:33-40) and CommunityAggregates.from_labels
//       (quality.py:71-79)                  -> build_members_and_aggregates: stable
//       sort of node ids by community; per-community sums in ascending node order
//       (bincount's sequential order, bit-exact even for real weights).
//   reverse_assignment (forest.py:70-80)   -> build_layout: children CSR (kids ascending)
//       plus a DFS pre-order layout of every community rooted at its smallest cycle node,
//       so that every assignment tail (detector.py:421-437) and every branch subtree
//       (detector.py:238-253) is one contiguous range.
//
// Fast path: cycles of the forest have length <= 2, so a node is on a cycle
// iff a[i] == i or a[a[i]] == i; every other node walks / pointer-jumps to its cycle.
// Arbitrary functional graphs (longer cycles) fall back to the reference's pointer
// doubling, so extract_components keeps its full contract.
#include "slm_internal.cuh"

#define GS_LOOP(i, n)                                                                      \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n);              \
         i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_cyc2(const int32_t *a, int64_t n, uint8_t *c2) {
    GS_LOOP(i, n) {
        int32_t x = a[i];
        c2[i] = (x == i) || (a[x] == i);
    }
}

__global__ void k_walk(const int32_t *a, const uint8_t *c2, int64_t n, int cap, int32_t *root,
                       int32_t *fail) {
    GS_LOOP(i, n) {
        int32_t x = (int32_t)i;
        int s = 0;
        while (!c2[x] && s < cap) {
            x = a[x];
            s++;
        }
        if (c2[x]) root[i] = x;
        else {
            root[i] = -1;
            *fail = 1;
        }
    }
}

__global__ void k_jump_init(const int32_t *a, const uint8_t *c2, const int32_t *root, int64_t n,
                            int32_t *r) {
    GS_LOOP(i, n) r[i] = root[i] >= 0 ? root[i] : (c2[i] ? (int32_t)i : a[i]);
}

__global__ void k_jump(const int32_t *rin, int64_t n, int32_t *rout, int32_t *changed) {
    GS_LOOP(i, n) {
        int32_t x = rin[i], y = rin[x];
        rout[i] = y;
        if (y != x) *changed = 1;
    }
}

__global__ void k_key_from_root(const int32_t *a, const int32_t *root, const uint8_t *c2,
                                int64_t n, int32_t *key, uint8_t *on_cycle, int32_t *bad) {
    GS_LOOP(i, n) {
        int32_t r = root[i];
        if (!c2[r]) *bad = 1;
        int32_t ar = a[r];
        key[i] = ar < r ? ar : r;
        on_cycle[i] = c2[i];
    }
}

// general path (forest.py:51-65): f = a^(2^k), on_cycle[f] = 1, minv propagation
__global__ void k_copy_i32(const int32_t *x, int64_t n, int32_t *y) { GS_LOOP(i, n) y[i] = x[i]; }
__global__ void k_square(const int32_t *f, int64_t n, int32_t *g) { GS_LOOP(i, n) g[i] = f[f[i]]; }
__global__ void k_mark_cycle(const int32_t *f, int64_t n, uint8_t *on_cycle) {
    GS_LOOP(i, n) on_cycle[f[i]] = 1;
}
__global__ void k_minv_step(const int32_t *minv, const int32_t *hop, int64_t n, int32_t *minv2,
                            int32_t *hop2) {
    GS_LOOP(i, n) {
        int32_t h = hop[i];
        int32_t v = minv[i], w = minv[h];
        minv2[i] = w < v ? w : v;
        hop2[i] = hop[h];
    }
}

__global__ void k_fill_i32(int32_t *x, int64_t n, int32_t v) { GS_LOOP(i, n) x[i] = v; }

__global__ void k_first_occ(const int32_t *key, int64_t n, int32_t *first) {
    // a hub component has millions of members: skip the same-address atomic once a smaller
    // member is already recorded (a stale read only costs an extra atomic)
    GS_LOOP(i, n) {
        const int32_t k = key[i];
        if ((int32_t)i < *(volatile int32_t *)&first[k]) atomicMin(&first[k], (int32_t)i);
    }
}
__global__ void k_head_flag(const int32_t *key, const int32_t *first, int64_t n, int32_t *h) {
    GS_LOOP(i, n) h[i] = (first[key[i]] == (int32_t)i) ? 1 : 0;
}
__global__ void k_assign_label(const int32_t *key, const int32_t *first, const int32_t *lab,
                               int64_t n, int32_t *comm, int32_t *croot) {
    GS_LOOP(i, n) {
        int32_t c = lab[first[key[i]]];
        comm[i] = c;
        if (key[i] == (int32_t)i) croot[c] = (int32_t)i;   // the smallest cycle node
    }
}

__global__ void k_iota(int32_t *x, int64_t n) { GS_LOOP(i, n) x[i] = (int32_t)i; }

// ptr[c] = first index of key c in a sorted array in which every key 0..nrows-1 occurs
__global__ void k_run_starts(const int32_t *sorted, int64_t m, int64_t nrows, int32_t *ptr) {
    GS_LOOP(i, m) if (i == 0 || sorted[i] != sorted[i - 1]) ptr[sorted[i]] = (int32_t)i;
    if (blockIdx.x == 0 && threadIdx.x == 0) ptr[nrows] = (int32_t)m;
}
__global__ void k_lb_one(const int32_t *sorted, int64_t m, int32_t key, int32_t *out) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (sorted[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    *out = (int32_t)lo;
}
__global__ void k_lb_ptr32(const int32_t *sorted, int64_t m, int64_t nrows, int32_t *ptr) {
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

// per-community sums of integer strengths: runs of equal community inside a warp's 32
// consecutive members are combined by a segmented shuffle scan, one atomic per run (exact:
// every partial sum is an integer below 2^53).  The community of the k-th member is the
// k-th sorted key, so the only gather is the node's interleaved strength pair (one sector);
// symmetric graphs accumulate s_out only (s_in is bitwise equal).
__global__ void k_comm_sums_runs(const int32_t *members, const int32_t *ksorted,
                                 const double2 *s2, int64_t n, bool sym, double *S_out,
                                 double *S_in) {
    const int lane = threadIdx.x & 31;
    for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31LL; b < n;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = b + lane;
        int32_t c = -1;
        double so = 0.0, si = 0.0;
        if (k < n) {
            c = ksorted[k];
            const double2 v = s2[members[k]];
            so = v.x;
            si = v.y;
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int32_t oc = __shfl_up_sync(0xffffffffu, c, off);
            const double oso = __shfl_up_sync(0xffffffffu, so, off);
            const double osi = sym ? 0.0 : __shfl_up_sync(0xffffffffu, si, off);
            if (lane >= off && oc == c) {
                so += oso;
                si += osi;
            }
        }
        const int32_t nc = __shfl_down_sync(0xffffffffu, c, 1);
        if (c >= 0 && (lane == 31 || nc != c)) {
            atomicAdd(&S_out[c], so);
            if (!sym) atomicAdd(&S_in[c], si);
        }
    }
}

// gather node strengths in member order (input of the segmented sums)
__global__ void k_gather_members(const int32_t *members, const double *s_out, const double *s_in,
                                 int64_t n, double *vo, double *vi) {
    GS_LOOP(k, n) {
        const int32_t x = members[k];
        vo[k] = s_out[x];
        vi[k] = s_in[x];
    }
}
__global__ void k_comm_finish(const int32_t *cptr, const double *S_out, double *S_in, bool sym,
                              int64_t nc, int32_t *count, double2 *S2, float *S1f, float2 *S2f) {
    GS_LOOP(c, nc) {
        const double so = S_out[c], si = sym ? so : S_in[c];
        if (sym) S_in[c] = so;
        S2[c] = make_double2(so, si);
        S1f[c] = (float)so;
        S2f[c] = make_float2((float)so, (float)si);
        count[c] = cptr[c + 1] - cptr[c];
    }
}

// per-community sums in ascending member order (bincount order, quality.py:76-78)
__global__ void k_comm_sums(const int32_t *cptr, const int32_t *members, const double *s_out,
                            const double *s_in, int64_t nc, double *S_out, double *S_in,
                            int32_t *count, double2 *S2, float *S1f, float2 *S2f) {
    GS_LOOP(c, nc) {
        double so = 0.0, si = 0.0;
        for (int32_t k = cptr[c]; k < cptr[c + 1]; k++) {
            int32_t x = members[k];
            so += s_out[x];
            si += s_in[x];
        }
        S_out[c] = so;
        S_in[c] = si;
        S2[c] = make_double2(so, si);
        S1f[c] = (float)so;
        S2f[c] = make_float2((float)so, (float)si);
        count[c] = cptr[c + 1] - cptr[c];
    }
}

__global__ void k_kid_flags(const int32_t *a, int64_t n, int32_t *f) {
    GS_LOOP(i, n) f[i] = a[i] != (int32_t)i;
}
__global__ void k_kid_compact(const int32_t *a, int64_t n, const int32_t *f, const int32_t *pos,
                              uint32_t *key, int32_t *node) {
    GS_LOOP(i, n) if (f[i]) {
        key[pos[i]] = (uint32_t)a[i];
        node[pos[i]] = (int32_t)i;
    }
}

// one thread per community: iterative DFS pre-order from the smallest cycle node
__global__ void k_dfs_layout(const int32_t *cptr, const int32_t *members, const uint8_t *on_cycle,
                             const int32_t *kptr, const int32_t *kids, int64_t nc, int32_t *order,
                             int32_t *pos, int32_t *sz, int32_t *stk_node, int32_t *stk_it) {
    GS_LOOP(c, nc) {
        int32_t base = cptr[c], end = cptr[c + 1];
        int32_t root = members[base];
        for (int32_t k = base; k < end; k++)
            if (on_cycle[members[k]]) {
                root = members[k];
                break;
            }
        int32_t cnt = 0, sp = 0;
        order[base] = root;
        pos[root] = 0;
        cnt = 1;
        stk_node[base] = root;
        stk_it[base] = kptr[root];
        sp = 1;
        while (sp > 0) {
            int32_t v = stk_node[base + sp - 1];
            int32_t it = stk_it[base + sp - 1];
            if (it < kptr[v + 1]) {
                int32_t k = kids[it];
                stk_it[base + sp - 1] = it + 1;
                if (k == root) continue;
                order[base + cnt] = k;
                pos[k] = cnt;
                cnt++;
                stk_node[base + sp] = k;
                stk_it[base + sp] = kptr[k];
                sp++;
            } else {
                sz[v] = cnt - pos[v];
                sp--;
            }
        }
    }
}

// ---- depth-parallel DFS layout (any community size; O(n * depth) work, depth is small)

__global__ void k_depth(const int32_t *a, const int32_t *comm, const int32_t *croot, int64_t n,
                        int cap, uint32_t *depth, int32_t *iota, int32_t *flags) {
    GS_LOOP(x, n) {
        const int32_t r = croot[comm[x]];
        int32_t y = (int32_t)x;
        int d = 0;
        while (y != r && d < cap) {
            y = a[y];
            d++;
        }
        if (y != r) atomicOr(&flags[0], 1);
        depth[x] = (uint32_t)d;
        iota[x] = (int32_t)x;
        const unsigned act = __activemask();
        const int dm = (int)__reduce_max_sync(act, (unsigned)d);   // one atomic per warp
        if ((threadIdx.x & 31) == __ffs(act) - 1) atomicMax(&flags[1], dm);
    }
}
__global__ void k_ones(int32_t *x, int64_t n) { GS_LOOP(i, n) x[i] = 1; }
__global__ void k_size_level(const int32_t *nodes, int64_t lo, int64_t hi, const int32_t *a,
                             int32_t *sz) {
    for (int64_t k = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < hi;
         k += (int64_t)gridDim.x * blockDim.x) {
        int32_t x = nodes[k];
        atomicAdd(&sz[a[x]], sz[x]);
    }
}
// small levels: every depth level in one launch (one CTA, a barrier between levels; lb[d] =
// first position of depth d in `nodes`).  The sizes are read around L1: the atomics of the
// level below land in L2.
__global__ void __launch_bounds__(1024) k_size_levels_cta(const int32_t *nodes, const int32_t *lb,
                                                          int maxd, const int32_t *a, int32_t *sz) {
    for (int d = maxd; d >= 1; d--) {
        const int lo = lb[d], hi = lb[d + 1];
        for (int k = lo + (int)threadIdx.x; k < hi; k += (int)blockDim.x) {
            const int32_t x = nodes[k];
            atomicAdd(&sz[a[x]], __ldcg(sz + x));
        }
        __syncthreads();
    }
}
__global__ void k_kid_vals(const int32_t *kids, int64_t nk, const int32_t *comm,
                           const int32_t *croot, const int32_t *sz, int32_t *val) {
    GS_LOOP(j, nk) {
        int32_t k = kids[j];
        val[j] = (croot[comm[k]] == k) ? 0 : sz[k];
    }
}
__global__ void k_kid_off(const int32_t *kids, const int32_t *ex, int64_t nk, int32_t *offp) {
    GS_LOOP(j, nk) offp[kids[j]] = 1 + ex[j];
}
__global__ void k_positions(const int32_t *a, const int32_t *comm, const int32_t *croot,
                            const int32_t *offp, const int32_t *cptr, int64_t n, int32_t *pos,
                            int32_t *order) {
    GS_LOOP(x, n) {
        const int32_t c = comm[x], r = croot[c];
        int32_t y = (int32_t)x, p = 0;
        while (y != r) {
            p += offp[y];
            y = a[y];
        }
        pos[x] = p;
        order[cptr[c] + p] = (int32_t)x;
    }
}

// ---------------------------------------------------------------------- host

void run_components(slm_ctx *ctx, Forest &F, int64_t n) {
    cudaStream_t s = ctx->stream;
    F.n = n;
    F.comm.resize(n);
    F.on_cycle.resize(n);
    if (n == 0) {
        F.n_comms = 0;
        return;
    }
    CTX_SCRATCH(DBuf<uint8_t>, c2);   // grow-only scratch kept across calls
    c2.resize(n);
    int32_t *root = ctx->i32a.resize(n);
    int32_t *key = ctx->i32b.resize(n);
    int32_t *flags = ctx->i32d.resize(4);
    CUDA_TRY(cudaMemsetAsync(flags, 0, 16, s));
    unsigned G = grid_for(n, 256);
    k_cyc2<<<G, 256, 0, s>>>(F.a.p, n, c2.p);
    k_walk<<<G, 256, 0, s>>>(F.a.p, c2.p, n, 64, root, flags);
    int32_t hf[4];
    CUDA_TRY(cudaMemcpyAsync(hf, flags, 16, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    bool general = false;
    if (hf[0]) {
        // deep trees: pointer jumping on root pointers
        int32_t *cur = ctx->i32c.resize(n);
        int32_t *nxt = root;
        k_jump_init<<<G, 256, 0, s>>>(F.a.p, c2.p, root, n, cur);
        int rounds = 0;
        for (;;) {
            CUDA_TRY(cudaMemsetAsync(flags + 1, 0, 4, s));
            k_jump<<<G, 256, 0, s>>>(cur, n, nxt, flags + 1);
            std::swap(cur, nxt);
            CUDA_TRY(cudaMemcpyAsync(hf, flags, 16, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            if (!hf[1] || ++rounds > 40) break;
        }
        if (cur != ctx->i32a.p)
            CUDA_TRY(cudaMemcpyAsync(ctx->i32a.p, cur, n * 4, cudaMemcpyDeviceToDevice, s));
        root = ctx->i32a.p;
        general = hf[1] != 0;
    }
    if (!general) {
        CUDA_TRY(cudaMemsetAsync(flags + 2, 0, 4, s));
        k_key_from_root<<<G, 256, 0, s>>>(F.a.p, root, c2.p, n, key, F.on_cycle.p, flags + 2);
        CUDA_TRY(cudaMemcpyAsync(hf, flags, 16, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        general = hf[2] != 0;   // some root is not on a <=2 cycle: longer cycles exist
    }
    if (general) {
        // the reference's pointer doubling (forest.py:51-65)
        int32_t *f = ctx->i32a.resize(n), *g = ctx->i32c.resize(n);
        k_copy_i32<<<G, 256, 0, s>>>(F.a.p, n, f);
        for (int64_t steps = 1; steps < n; steps *= 2) {
            k_square<<<G, 256, 0, s>>>(f, n, g);
            std::swap(f, g);
        }
        CUDA_TRY(cudaMemsetAsync(F.on_cycle.p, 0, n, s));
        k_mark_cycle<<<G, 256, 0, s>>>(f, n, F.on_cycle.p);
        CTX_SCRATCH(DBuf<int32_t>, hop);   // grow-only scratch kept across calls
        CTX_SCRATCH(DBuf<int32_t>, hop2);
        CTX_SCRATCH(DBuf<int32_t>, mv2);
        hop.resize(n);
        hop2.resize(n);
        mv2.resize(n);
        int32_t *minv = key;
        k_copy_i32<<<G, 256, 0, s>>>(f, n, minv);
        k_copy_i32<<<G, 256, 0, s>>>(F.a.p, n, hop.p);
        int32_t *m1 = minv, *m2 = mv2.p, *h1 = hop.p, *h2 = hop2.p;
        for (int64_t steps = 1; steps < n; steps *= 2) {
            k_minv_step<<<G, 256, 0, s>>>(m1, h1, n, m2, h2);
            std::swap(m1, m2);
            std::swap(h1, h2);
        }
        if (m1 != key) CUDA_TRY(cudaMemcpyAsync(key, m1, n * 4, cudaMemcpyDeviceToDevice, s));
    }
    // canonical labels ordered by smallest member
    int32_t *first = ctx->i32c.resize(n);
    k_fill_i32<<<G, 256, 0, s>>>(first, n, 0x7fffffff);
    k_first_occ<<<G, 256, 0, s>>>(key, n, first);
    CTX_SCRATCH(DBuf<int32_t>, h);   // grow-only scratch kept across calls
    CTX_SCRATCH(DBuf<int32_t>, lab);
    h.resize(n + 1);
    lab.resize(n + 1);
    CUDA_TRY(cudaMemsetAsync(h.p + n, 0, 4, s));
    k_head_flag<<<G, 256, 0, s>>>(key, first, n, h.p);
    dev_exclusive_sum<int32_t, int32_t>(ctx, h.p, lab.p, n + 1);
    F.croot.resize(n);
    k_assign_label<<<G, 256, 0, s>>>(key, first, lab.p, n, F.comm.p, F.croot.p);
    int32_t nc = 0;
    CUDA_TRY(cudaMemcpyAsync(&nc, lab.p + n, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    F.n_comms = nc;
    F.layout_valid = false;
    F.agg_valid = false;
}

void build_members_and_aggregates(slm_ctx *ctx, const LevelGraph &G, Forest &F) {
    cudaStream_t s = ctx->stream;
    int64_t n = F.n, nc = F.n_comms;
    F.members.resize(n);
    F.cptr.resize(nc + 1);
    F.S_out.resize(nc);
    F.S_in.resize(nc);
    F.S2.resize(nc);
    F.S1f.resize(nc);
    F.S2f.resize(nc);
    F.count.resize(nc);
    int32_t *iota = ctx->i32a.resize(n);
    int32_t *ksorted = ctx->i32b.resize(n);
    k_iota<<<grid_for(n, 256), 256, 0, s>>>(iota, n);
    if (n > 0)
        sort_pairs_u32_i32(ctx, (uint32_t *)F.comm.p, (uint32_t *)ksorted, iota, F.members.p, n,
                           bits_for(nc + 1));
    k_run_starts<<<grid_for(n, 256), 256, 0, s>>>(ksorted, n, nc, F.cptr.p);
    // segmented sums over the member-ordered strengths (exact for integer weights in any
    // order; CUB's fixed reduction tree keeps real-valued sums deterministic)
    if (!G.integral) {
        // real weights: sequential per-community sums in node order (numpy bincount order)
        k_comm_sums<<<grid_for(nc, 128), 128, 0, s>>>(F.cptr.p, F.members.p, G.s_out.p, G.s_in.p,
                                                      nc, F.S_out.p, F.S_in.p, F.count.p, F.S2.p,
                                                      F.S1f.p, F.S2f.p);
        F.agg_valid = true;
        return;
    }
    CUDA_TRY(cudaMemsetAsync(F.S_out.p, 0, nc * 8, s));
    if (!G.sym) CUDA_TRY(cudaMemsetAsync(F.S_in.p, 0, nc * 8, s));
    k_comm_sums_runs<<<grid_for(n, 256), 256, 0, s>>>(F.members.p, ksorted, G.s2.p, n, G.sym,
                                                       F.S_out.p, F.S_in.p);
    k_comm_finish<<<grid_for(nc, 256), 256, 0, s>>>(F.cptr.p, F.S_out.p, F.S_in.p, G.sym, nc,
                                                    F.count.p,
                                                    F.S2.p, F.S1f.p, F.S2f.p);
    F.agg_valid = true;
}

void build_layout(slm_ctx *ctx, Forest &F) {
    cudaStream_t s = ctx->stream;
    int64_t n = F.n, nc = F.n_comms;
    F.kptr.resize(n + 1);
    F.kids.resize(n);
    F.order.resize(n);
    F.pos.resize(n);
    F.sz.resize(n);
    uint32_t *kk = (uint32_t *)ctx->i32a.resize(n);
    uint32_t *ks = (uint32_t *)ctx->i32b.resize(n);
    int32_t *iota = ctx->i32c.resize(n);
    // the children lists: nodes with a[i] != i, stably sorted by parent.  They are compacted
    // first, so the sort runs on parent ids alone (bits_for(n) bits: 3 passes at n = 2^24,
    // where keys with a sentinel for self-assigned nodes would need a fourth)
    {
        CTX_SCRATCH(DBuf<int32_t>, kf);
        CTX_SCRATCH(DBuf<int32_t>, kpos);
        kf.resize(n + 1);
        kpos.resize(n + 1);
        CUDA_TRY(cudaMemsetAsync(kf.p + n, 0, 4, s));
        k_kid_flags<<<grid_for(n, 256), 256, 0, s>>>(F.a.p, n, kf.p);
        dev_exclusive_sum<int32_t, int32_t>(ctx, kf.p, kpos.p, n + 1);
        k_kid_compact<<<grid_for(n, 256), 256, 0, s>>>(F.a.p, n, kf.p, kpos.p, kk, iota);
        int32_t nkids = 0;
        CUDA_TRY(cudaMemcpyAsync(&nkids, kpos.p + n, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        if (nkids > 0) sort_pairs_u32_i32(ctx, kk, ks, iota, F.kids.p, nkids, bits_for(n));
        // only kptr[n] (the number of kids) is needed unless the DFS fallback below runs
        CUDA_TRY(cudaMemcpyAsync(F.kptr.p + n, kpos.p + n, 4, cudaMemcpyDeviceToDevice, s));
    }
    // depth of every node below its community root (parent = a[x])
    int32_t *flags = ctx->i32d.resize(2);
    CUDA_TRY(cudaMemsetAsync(flags, 0, 8, s));
    CTX_SCRATCH(DBuf<uint32_t>, depth);   // grow-only scratch kept across calls
    CTX_SCRATCH(DBuf<uint32_t>, depth_sorted);
    CTX_SCRATCH(DBuf<int32_t>, by_depth);   // grow-only scratch kept across calls
    depth.resize(n);
    depth_sorted.resize(n);
    by_depth.resize(n);
    int32_t *iota2 = ctx->i32a.resize(n);
    k_depth<<<grid_for(n, 256), 256, 0, s>>>(F.a.p, F.comm.p, F.croot.p, n, 4096, depth.p,
                                              iota2, flags);
    int32_t hf[2];
    int32_t nk = 0;
    CUDA_TRY(cudaMemcpyAsync(hf, flags, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&nk, F.kptr.p + n, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    const int maxd = hf[1];
    if (hf[0]) {
        // pathological depth (> 4096): sequential DFS per community (needs the kids pointers)
        k_lb_ptr32<<<grid_for(n + 1, 256), 256, 0, s>>>((const int32_t *)ks, nk, n, F.kptr.p);
        int32_t *stk_node = ctx->i32a.resize(n);
        CTX_SCRATCH(DBuf<int32_t>, stk_it);   // grow-only scratch kept across calls
        stk_it.resize(n);
        k_dfs_layout<<<grid_for(nc, 64), 64, 0, s>>>(F.cptr.p, F.members.p, F.on_cycle.p, F.kptr.p,
                                                     F.kids.p, nc, F.order.p, F.pos.p, F.sz.p,
                                                     stk_node, stk_it.p);
        CUDA_TRY(cudaGetLastError());
        F.layout_valid = true;
        return;
    }
    // subtree sizes bottom-up, one launch per depth level
    if (n > 0)
        sort_pairs_u32_i32(ctx, depth.p, depth_sorted.p, iota2, by_depth.p, n, bits_for(maxd + 2));
    CTX_SCRATCH(DBuf<int32_t>, lb);   // grow-only scratch kept across calls
    lb.resize(maxd + 2);
    k_run_starts<<<grid_for(n, 256), 256, 0, s>>>((const int32_t *)depth_sorted.p, n, maxd + 1, lb.p);
    k_ones<<<grid_for(n, 256), 256, 0, s>>>(F.sz.p, n);
    if (n <= 32768) {
        // launch-bound sizes: one CTA walks the depth levels (no host copy of the bounds)
        if (maxd >= 1)
            k_size_levels_cta<<<1, 1024, 0, s>>>(by_depth.p, lb.p, maxd, F.a.p, F.sz.p);
    } else {
        std::vector<int64_t> lvl(maxd + 2, 0);
        std::vector<int32_t> h(maxd + 2);
        CUDA_TRY(cudaMemcpyAsync(h.data(), lb.p, (maxd + 2) * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        for (int d = 0; d <= maxd + 1; d++) lvl[d] = h[d];
        for (int d = maxd; d >= 1; d--) {
            int64_t lo = lvl[d], hi = lvl[d + 1];
            if (hi > lo)
                k_size_level<<<grid_for(hi - lo, 256), 256, 0, s>>>(by_depth.p, lo, hi, F.a.p, F.sz.p);
        }
    }
    // offsets among siblings (kids ascending, the root never a kid) and pre-order positions
    CTX_SCRATCH(DBuf<int32_t>, val);   // grow-only scratch kept across calls
    CTX_SCRATCH(DBuf<int32_t>, ex);
    CTX_SCRATCH(DBuf<int32_t>, offp);
    val.resize(nk);
    ex.resize(nk);
    offp.resize(n);
    if (nk > 0) {
        k_kid_vals<<<grid_for(nk, 256), 256, 0, s>>>(F.kids.p, nk, F.comm.p, F.croot.p, F.sz.p, val.p);
        dev_exclusive_sum_by_key(ctx, (const uint32_t *)ks, val.p, ex.p, (int64_t)nk);
        k_kid_off<<<grid_for(nk, 256), 256, 0, s>>>(F.kids.p, ex.p, nk, offp.p);
    }
    k_positions<<<grid_for(n, 256), 256, 0, s>>>(F.a.p, F.comm.p, F.croot.p, offp.p, F.cptr.p, n,
                                                  F.pos.p, F.order.p);
    CUDA_TRY(cudaGetLastError());
    F.layout_valid = true;
}

void forest_refresh(slm_ctx *ctx, const LevelGraph &G, Forest &F) {
    phase_mark(ctx, -1);
    run_components(ctx, F, G.n);
    phase_mark(ctx, PH_REFRESH_COMP);
    build_members_and_aggregates(ctx, G, F);
    phase_mark(ctx, PH_REFRESH_AGG);
    build_layout(ctx, F);
    phase_mark(ctx, PH_REFRESH_LAYOUT);
    F.version++;
}

// a kernel of this translation unit (module preloading, slm_capi.cu preload_modules)
const void *slm_anchor_forest() { return (const void *)k_cyc2; }
