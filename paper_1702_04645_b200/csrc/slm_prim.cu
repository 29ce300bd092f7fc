// slm_prim.cu -- the library's own device primitives: single-pass prefix scans and a stable
// onesweep LSD radix sort (no CUB).  They carry the sort + segmented-reduce of the CSR build
// and the aggregation (Graph.from_edges / aggregate: graph.py:97-116, 266-280 -- numpy's
// stable lexsort, reduceat offsets and bincount/cumsum pointers), the forest's member and
// child lists, the commit timelines and the POSITIVE layouts.
//
// Scan.  One launch: every CTA takes the next tile id from an atomic counter (so a tile only
// ever waits on tiles that are already running), reduces its tile, publishes the aggregate,
// then walks back over its predecessors' published aggregates / inclusive prefixes
// ("decoupled look-back") until it meets an inclusive prefix, publishes its own inclusive
// prefix and writes the tile.  The segmented form (exclusive sum restarting at every key
// change) scans (value, head) pairs with the segmented operator.  Tiles combine in a fixed
// order, so results are deterministic (for fp64 operands too).
//
// Radix sort.  8-bit digits, least significant first; one histogram kernel counts the
// digits of every pass in a single read of the keys, then one onesweep kernel per pass:
//   - a tile of 16 keys per thread is ranked warp by warp: each warp walks its contiguous
//     segment in input order in 32-key chunks, __match_any_sync groups equal digits, the
//     group leader bumps the warp's private digit counter (stable by construction);
//   - per digit, warp offsets and the tile count, then the tile's global offset by
//     decoupled look-back over the preceding tiles (one 64-bit {flag, count} word per
//     (tile, digit));
//   - keys (then values) are staged in shared memory in digit order and written out from
//     there, so every digit's run leaves the CTA as contiguous stores.
#include "slm_internal.cuh"
#include <type_traits>

namespace {

constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_ITEMS;

__device__ __forceinline__ int ld_flag(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_flag(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// scan state: value plus (segmented form) "a segment starts inside" flag
template <class T, bool SEG>
struct SS {
    T v;
    int h;
};
template <class T, bool SEG>
__device__ __forceinline__ SS<T, SEG> sop(SS<T, SEG> a, SS<T, SEG> b) {
    if (SEG && b.h) return b;
    return {a.v + b.v, a.h | b.h};
}

template <class T, bool SEG>
__device__ __forceinline__ SS<T, SEG> shfl_up_ss(SS<T, SEG> x, int d) {
    SS<T, SEG> y;
    y.v = __shfl_up_sync(0xffffffffu, x.v, d);
    y.h = __shfl_up_sync(0xffffffffu, x.h, d);
    return y;
}

// tile status: flag 0 = not ready, 1 = aggregate, 2 = inclusive prefix
template <class T>
struct ScanStatus {
    int *flag;
    T *agg, *inc;
    int *hagg, *hinc;
    unsigned *ticket;
};

// per-thread items, thread/warp/block inclusive scan of a tile (shared by both scan forms)
template <class TI, class TO, bool SEG>
struct TileScan {
    SS<TO, SEG> x[SCAN_ITEMS];
    SS<TO, SEG> w;   // warp-inclusive scan of the thread totals
    __device__ __forceinline__ void load(const TI *in, const uint32_t *keys, int64_t n,
                                         int64_t base) {
#pragma unroll
        for (int i = 0; i < SCAN_ITEMS; i++) {
            const int64_t k = base + i;
            x[i].v = k < n ? (TO)in[k] : (TO)0;
            x[i].h = 0;
            if (SEG && k < n) x[i].h = (k == 0 || keys[k] != keys[k - 1]) ? 1 : 0;
        }
    }
    // returns the tile aggregate (valid in every thread after the call); s_warp gets the
    // inclusive scan over warps
    __device__ __forceinline__ SS<TO, SEG> reduce(SS<TO, SEG> *s_warp) {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        SS<TO, SEG> t = x[0];
#pragma unroll
        for (int i = 1; i < SCAN_ITEMS; i++) t = sop<TO, SEG>(t, x[i]);
        w = t;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            SS<TO, SEG> y = shfl_up_ss<TO, SEG>(w, d);
            if (lane >= d) w = sop<TO, SEG>(y, w);
        }
        if (lane == 31) s_warp[wid] = w;
        __syncthreads();
        if (wid == 0) {
            SS<TO, SEG> v = lane < SCAN_BLOCK / 32 ? s_warp[lane] : SS<TO, SEG>{(TO)0, 0};
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                SS<TO, SEG> y = shfl_up_ss<TO, SEG>(v, d);
                if (lane >= d) v = sop<TO, SEG>(y, v);
            }
            if (lane < SCAN_BLOCK / 32) s_warp[lane] = v;
        }
        __syncthreads();
        return s_warp[SCAN_BLOCK / 32 - 1];
    }
    // write the exclusive scan given the tile's exclusive prefix
    __device__ __forceinline__ void write(TO *out, int64_t n, int64_t base, SS<TO, SEG> prefix,
                                          const SS<TO, SEG> *s_warp) {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        SS<TO, SEG> run = prefix;
        if (wid > 0) run = sop<TO, SEG>(run, s_warp[wid - 1]);
        SS<TO, SEG> wl = shfl_up_ss<TO, SEG>(w, 1);
        if (lane > 0) run = sop<TO, SEG>(run, wl);
#pragma unroll
        for (int i = 0; i < SCAN_ITEMS; i++) {
            const int64_t k = base + i;
            if (SEG && x[i].h) run = SS<TO, SEG>{(TO)0, 1};
            if (k < n) out[k] = run.v;
            run = sop<TO, SEG>(run, SS<TO, SEG>{x[i].v, 0});
        }
    }
};

// single pass, integer operands (exact, so the look-back's grouping is immaterial): warp 0
// looks back 32 predecessor tiles at a time; the nearest one holding an inclusive prefix
// (or, segmented, a segment start) ends the walk
template <class TI, class TO, bool SEG>
__global__ void __launch_bounds__(SCAN_BLOCK) k_scan(const TI *in, TO *out, const uint32_t *keys,
                                                     int64_t n, ScanStatus<TO> st) {
    __shared__ unsigned s_tile;
    __shared__ SS<TO, SEG> s_warp[SCAN_BLOCK / 32];
    __shared__ SS<TO, SEG> s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(st.ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    TileScan<TI, TO, SEG> T;
    T.load(in, keys, n, base);
    const SS<TO, SEG> agg = T.reduce(s_warp);
    if (wid == 0) {
        if (tile == 0) {
            if (lane == 0) {
                st.inc[0] = agg.v;
                st.hinc[0] = agg.h;
                st_flag(st.flag, 2);
                s_prefix = SS<TO, SEG>{(TO)0, 0};
            }
        } else {
            if (lane == 0) {
                st.agg[tile] = agg.v;
                st.hagg[tile] = agg.h;
                st_flag(st.flag + tile, 1);
            }
            TO pv = 0;
            int ph = 0;
            for (int64_t p = tile - 1;; p -= 32) {
                const int64_t q = p - lane;
                int f = q >= 0 ? ld_flag(st.flag + q) : 2;
                while (__any_sync(0xffffffffu, f == 0))
                    if (f == 0) f = ld_flag(st.flag + q);
                TO v = 0;
                int h = 0;
                if (q >= 0) {
                    v = f == 2 ? st.inc[q] : st.agg[q];
                    if (SEG) h = f == 2 ? st.hinc[q] : st.hagg[q];
                }
                const unsigned stop = __ballot_sync(0xffffffffu, f == 2 || (SEG && h));
                const int last = stop ? __ffs(stop) - 1 : 31;   // lanes 0..last contribute
                TO sum = lane <= last ? v : (TO)0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                const int hl = __shfl_sync(0xffffffffu, h, last);
                // earlier window (+) later prefix: a segment start in the later part wins
                if (!ph) {
                    pv += sum;
                    ph = SEG ? hl : 0;
                }
                if (stop) break;
            }
            if (lane == 0) {
                const SS<TO, SEG> pre{pv, ph};
                const SS<TO, SEG> inc = sop<TO, SEG>(pre, agg);
                st.inc[tile] = inc.v;
                st.hinc[tile] = inc.h;
                st_flag(st.flag + tile, 2);
                s_prefix = pre;
            }
        }
    }
    __syncthreads();
    T.write(out, n, base, s_prefix, s_warp);
}

// deterministic reduce-then-scan for fp64 operands (the look-back's grouping would make
// the rounding depend on timing): tile sums, one CTA scans them in order, tiles rescan
template <class TI, class T>
__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_reduce(const TI *in, int64_t n, T *tsum) {
    __shared__ SS<T, false> s_warp[SCAN_BLOCK / 32];
    TileScan<TI, T, false> S;
    const int64_t base = blockIdx.x * (int64_t)SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    S.load(in, nullptr, n, base);
    const SS<T, false> agg = S.reduce(s_warp);
    if (threadIdx.x == 0) tsum[blockIdx.x] = agg.v;
}
template <class T>
__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_tiles(T *tsum, int64_t nt) {
    __shared__ SS<T, false> s_warp[SCAN_BLOCK / 32];
    __shared__ T carry;
    if (threadIdx.x == 0) carry = (T)0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < nt; b0 += SCAN_TILE) {
        TileScan<T, T, false> S;
        const int64_t base = b0 + (int64_t)threadIdx.x * SCAN_ITEMS;
        S.load(tsum, nullptr, nt, base);
        const SS<T, false> agg = S.reduce(s_warp);
        const T c = carry;
        S.write(tsum, nt, base, SS<T, false>{c, 0}, s_warp);
        __syncthreads();
        if (threadIdx.x == 0) carry = c + agg.v;
        __syncthreads();
    }
}
template <class TI, class T>
__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_down(const TI *in, T *out, int64_t n,
                                                          const T *tpre) {
    __shared__ SS<T, false> s_warp[SCAN_BLOCK / 32];
    TileScan<TI, T, false> S;
    const int64_t base = blockIdx.x * (int64_t)SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    S.load(in, nullptr, n, base);
    S.reduce(s_warp);
    // tpre == nullptr: a single tile, nothing before it
    S.write(out, n, base, SS<T, false>{tpre ? tpre[blockIdx.x] : T(0), 0}, s_warp);
}

template <class TO>
void scan_launch_status(slm_ctx *ctx, int64_t ntiles, ScanStatus<TO> &st) {
    // [ticket | flags (ntiles) | hagg | hinc | agg | inc]
    const size_t ib = (size_t)(3 * ntiles + 4) * sizeof(int);
    const size_t vb = (size_t)(2 * ntiles) * sizeof(TO);
    ctx->tmp.resize(ib + vb + 16);
    char *p = (char *)ctx->tmp.p;
    st.ticket = (unsigned *)p;
    st.flag = (int *)p + 4;
    st.hagg = st.flag + ntiles;
    st.hinc = st.hagg + ntiles;
    char *q = p + ((ib + 15) & ~(size_t)15);
    st.agg = (TO *)q;
    st.inc = st.agg + ntiles;
    CUDA_TRY(cudaMemsetAsync(p, 0, (size_t)(ntiles + 4) * sizeof(int), ctx->stream));
}

template <class TI, class TO, bool SEG>
void scan_run(slm_ctx *ctx, const TI *in, TO *out, const uint32_t *keys, int64_t n) {
    if (n <= 0) return;
    const int64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (!SEG && ntiles == 1) {
        // one tile: the down-sweep kernel alone (the same arithmetic with a zero prefix) --
        // small levels are launch-bound, so every kernel saved counts
        k_scan_down<TI, TO><<<1, SCAN_BLOCK, 0, ctx->stream>>>(in, out, n, (const TO *)nullptr);
    } else if (!SEG) {
        // reduce-then-scan: tile sums, one CTA scans them in order, tiles rescan.  Fixed
        // order (deterministic fp64 rounding), and no look-back chain across the ~1,000
        // tiles resident at once (the single-pass form below is kept for the segmented scan)
        ctx->tmp.resize(ntiles * sizeof(TO));
        TO *tsum = (TO *)ctx->tmp.p;
        k_scan_reduce<TI, TO><<<(unsigned)ntiles, SCAN_BLOCK, 0, ctx->stream>>>(in, n, tsum);
        k_scan_tiles<TO><<<1, SCAN_BLOCK, 0, ctx->stream>>>(tsum, ntiles);
        k_scan_down<TI, TO><<<(unsigned)ntiles, SCAN_BLOCK, 0, ctx->stream>>>(in, out, n, tsum);
    } else {
        ScanStatus<TO> st;
        scan_launch_status<TO>(ctx, ntiles, st);
        k_scan<TI, TO, SEG><<<(unsigned)ntiles, SCAN_BLOCK, 0, ctx->stream>>>(in, out, keys, n, st);
    }
    CUDA_TRY(cudaGetLastError());
}

// ------------------------------------------------------------------- radix sort

constexpr int RS_BLOCK = 512;
constexpr int RS_WARPS = RS_BLOCK / 32;
constexpr int RS_ITEMS = 12;
constexpr int RS_TILE = RS_BLOCK * RS_ITEMS;
constexpr int RS_MAXP = 8;

// digit of pass p: bits [begin + 8p, min(begin + 8p + 8, end)) (bits at or above end_bit
// are ignored, as a sort "by bits [begin, end)" must)
__device__ __forceinline__ unsigned pass_mask(int shift, int end_bit) {
    const int w = end_bit - shift;
    return w >= 8 ? 255u : ((1u << w) - 1u);
}

template <class K>
__global__ void __launch_bounds__(256) k_rs_hist(const K *keys, int64_t n, int begin_bit, int np,
                                                 int end_bit, unsigned long long *hist) {
    __shared__ unsigned sh[RS_MAXP][256];
    for (int i = threadIdx.x; i < RS_MAXP * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const K k = keys[i];
        for (int p = 0; p < np; p++) {
            const int sh_ = begin_bit + 8 * p;
            const unsigned d = (unsigned)(k >> sh_) & pass_mask(sh_, end_bit);
            atomicAdd(&sh[p][d], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < np * 256; i += blockDim.x) {
        const unsigned v = (&sh[0][0])[i];
        if (v) atomicAdd(hist + i, (unsigned long long)v);
    }
}

// exclusive scan of each pass's 256 digit counts (one CTA per pass)
__global__ void k_rs_hist_scan(unsigned long long *hist) {
    __shared__ unsigned long long s[256];
    unsigned long long *h = hist + blockIdx.x * 256;
    const int t = threadIdx.x;
    s[t] = h[t];
    __syncthreads();
    for (int d = 1; d < 256; d <<= 1) {
        unsigned long long v = t >= d ? s[t - d] : 0ull;
        __syncthreads();
        s[t] += v;
        __syncthreads();
    }
    h[t] = s[t] - h[t];
}

constexpr unsigned long long RS_AGG = 1ull << 62, RS_INC = 2ull << 62, RS_VAL = RS_AGG - 1;

__device__ __forceinline__ unsigned long long ld_status(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_status(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <class K, class V>
__global__ void __launch_bounds__(RS_BLOCK, 2) k_rs_onesweep(const K *kin, K *kout, const V *vin,
                                                          V *vout, int64_t n, int shift,
                                                          unsigned dmask,
                                                          const unsigned long long *dbase,
                                                          unsigned long long *status,
                                                          unsigned *ticket,
                                                          const int64_t *toff, int64_t ntiles) {
    extern __shared__ __align__(16) unsigned char rs_smem[];
    unsigned *wcnt = (unsigned *)rs_smem;                                   // [WARPS][256]
    unsigned long long *dest = (unsigned long long *)(wcnt + RS_WARPS * 256);   // [256]
    unsigned *tstart = (unsigned *)(dest + 256);                            // [256]
    unsigned char *sdig = (unsigned char *)(tstart + 256);                  // [TILE]
    K *sk = (K *)(sdig + RS_TILE);                                          // [TILE] (keys, then values)
    __shared__ unsigned s_tile;
    __shared__ unsigned s_hist[256];
    // reduce-then-scan mode (toff != nullptr): the tile's offsets per digit are known,
    // tile = blockIdx.x; onesweep mode: tiles in ticket order with decoupled look-back
    // single-tile mode (dbase == nullptr, toff == nullptr): the staged digit order is the
    // output order -- no histogram, no status words, no ticket
    const bool single = !toff && !dbase;
    if (threadIdx.x == 0) s_tile = (toff || single) ? blockIdx.x : atomicAdd(ticket, 1u);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i = lane; i < 256; i += 32) {
        wcnt[wid * 256 + i] = 0;
        ((unsigned *)sk)[wid * 256 + i] = 0;   // per-warp digit masks of the ranking
    }
    if (threadIdx.x < 256) s_hist[threadIdx.x] = 0;
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t t0 = tile * RS_TILE;
    const int64_t wb = t0 + (int64_t)wid * 32 * RS_ITEMS;
    K key[RS_ITEMS];
    unsigned pos[RS_ITEMS];
    // 4-byte values are loaded with the keys (their latency overlaps the ranking)
    constexpr bool VPRE = sizeof(V) == 4;
    V val[VPRE ? RS_ITEMS : 1];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < RS_ITEMS; i++) {
        const int64_t idx = wb + i * 32 + lane;
        key[i] = idx < n ? kin[idx] : (K)0;
        if (VPRE && vin) val[VPRE ? i : 0] = idx < n ? vin[idx] : (V)0;
    }
    // the tile's digit counts first, published at once, so that the tiles behind this one
    // find them during their look-back while this tile is still ranking its keys
    if (!toff && !single) {
#pragma unroll
        for (int i = 0; i < RS_ITEMS; i++)
            if (wb + i * 32 + lane < n) atomicAdd(&s_hist[(unsigned)(key[i] >> shift) & dmask], 1u);
        __syncthreads();
        if (threadIdx.x < 256)
            st_status(status + tile * 256 + threadIdx.x,
                      (tile == 0 ? RS_INC : RS_AGG) | s_hist[threadIdx.x]);
    }
    // peers of equal digit inside a 32-key chunk: every lane ORs its bit into the warp's
    // per-digit mask (shared memory, the staging area before it is used), then reads it
    // back; the lowest peer advances the warp's digit counter and clears the mask
    // (cheaper than __match_any_sync)
    unsigned *msk = (unsigned *)sk + wid * 256;
#pragma unroll
    for (int i = 0; i < RS_ITEMS; i++) {
        const bool ok = wb + i * 32 + lane < n;
        const unsigned d = (unsigned)(key[i] >> shift) & dmask;
        if (ok) atomicOr(&msk[d], 1u << lane);
        __syncwarp();
        const unsigned m = ok ? msk[d] : 0u;
        __syncwarp();
        const int leader = ok ? __ffs(m) - 1 : lane;
        unsigned base = 0;
        if (ok && lane == leader) {
            base = wcnt[wid * 256 + d];
            wcnt[wid * 256 + d] = base + __popc(m);
            msk[d] = 0u;
        }
        base = __shfl_sync(0xffffffffu, base, leader);
        __syncwarp();
        pos[i] = ok ? ((base + __popc(m & lt)) | (d << 24)) : 0xffffffffu;   // rank | digit
    }
    __syncthreads();
    // per digit: warp offsets, tile count, tile start in digit order
    unsigned cnt = 0;
    if (threadIdx.x < 256) {
        const int d = threadIdx.x;
        for (int w = 0; w < RS_WARPS; w++) {
            const unsigned c = wcnt[w * 256 + d];
            wcnt[w * 256 + d] = cnt;
            cnt += c;
        }
        // look back for the global prefix of this digit (the count was published above)
        unsigned long long *mine = status + tile * 256 + d;
        unsigned long long excl = 0;
        if (toff) {
            dest[d] = (unsigned long long)toff[(int64_t)d * ntiles + tile];
        } else if (tile != 0 && !single) {
            // 8 predecessors per step with independent loads: the walk costs one memory
            // latency per 8 tiles, not per tile
            for (int64_t p = tile - 1; p >= 0;) {
                constexpr int LB = 8;
                unsigned long long sv[LB];
#pragma unroll
                for (int k = 0; k < LB; k++)
                    sv[k] = p - k >= 0 ? ld_status(status + (p - k) * 256 + d) : RS_INC;
                int k = 0;
                bool done = false;
                for (; k < LB; k++) {
                    if ((sv[k] >> 62) == 0) break;           // not published yet: reload
                    excl += sv[k] & RS_VAL;
                    if ((sv[k] >> 62) == 2) {
                        done = true;
                        break;
                    }
                }
                if (done) break;
                p -= k;
            }
            st_status(mine, RS_INC | (excl + cnt));
        }
        if (!toff && !single) dest[d] = dbase[d] + excl;
    }
    // tile start of every digit in digit order: exclusive scan of cnt over 256 threads
    {
        __shared__ unsigned s_w[8];
        unsigned v = cnt;
        if (threadIdx.x < 256) {
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += y;
            }
            if (lane == 31) s_w[wid] = v;
        }
        __syncthreads();
        if (threadIdx.x < 256) {
            unsigned off = 0;
            for (int w = 0; w < wid; w++) off += s_w[w];
            tstart[threadIdx.x] = off + v - cnt;
            if (single) dest[threadIdx.x] = off + v - cnt;
        }
    }
    __syncthreads();
    // stage keys in digit order
    const int64_t nt = min((int64_t)RS_TILE, n - t0);
#pragma unroll
    for (int i = 0; i < RS_ITEMS; i++) {
        if (pos[i] == 0xffffffffu) continue;
        const unsigned d = pos[i] >> 24;
        const unsigned lp = tstart[d] + wcnt[wid * 256 + d] + (pos[i] & 0xffffffu);
        pos[i] = lp;
        sk[lp] = key[i];
        sdig[lp] = (unsigned char)d;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nt; j += RS_BLOCK) {
        const unsigned d = sdig[j];
        kout[dest[d] + (j - tstart[d])] = sk[j];
    }
    if (vin) {
        __syncthreads();
        V *sv = (V *)sk;
#pragma unroll
        for (int i = 0; i < RS_ITEMS; i++) {
            const int64_t idx = wb + i * 32 + lane;
            if (idx < n) sv[pos[i]] = VPRE ? val[VPRE ? i : 0] : vin[idx];
        }
        __syncthreads();
        for (int j = threadIdx.x; j < nt; j += RS_BLOCK) {
            const unsigned d = sdig[j];
            vout[dest[d] + (j - tstart[d])] = sv[j];
        }
    }
}

// reduce-then-scan upsweep: per tile, the digit counts of this pass, digit-major
// (cnt[d * ntiles + tile]); their exclusive scan is every (digit, tile)'s output offset
template <class K>
__global__ void __launch_bounds__(RS_BLOCK) k_rs_tilehist(const K *kin, int64_t n, int shift,
                                                        unsigned dmask, int64_t ntiles,
                                                        int32_t *cnt) {
    __shared__ unsigned h[256];
    if (threadIdx.x < 256) h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t t0 = blockIdx.x * (int64_t)RS_TILE;
#pragma unroll 4
    for (int i = 0; i < RS_ITEMS; i++) {
        const int64_t idx = t0 + (int64_t)i * RS_BLOCK + threadIdx.x;
        if (idx < n) atomicAdd(&h[(unsigned)(kin[idx] >> shift) & dmask], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 256) cnt[(int64_t)threadIdx.x * ntiles + blockIdx.x] = (int32_t)h[threadIdx.x];
}

template <class K, class V>
size_t rs_smem_bytes() {
    const size_t kv = sizeof(K) > sizeof(V) ? sizeof(K) : sizeof(V);
    return RS_WARPS * 256 * 4 + 256 * 8 + 256 * 4 + RS_TILE + RS_TILE * kv;
}

// stable sort of (kin, vin) by bits [begin_bit, end_bit) into (kout, vout); kalt / valt are
// n-element scratch; vin == nullptr sorts keys only.  Inputs are left untouched.
template <class K, class V>
void radix_sort_impl(slm_ctx *ctx, const K *kin, K *kout, const V *vin, V *vout, K *kalt, V *valt,
                     int64_t n, int begin_bit, int end_bit) {
    cudaStream_t s = ctx->stream;
    if (n <= 0) return;
    const int np = end_bit > begin_bit ? (end_bit - begin_bit + 7) / 8 : 0;
    if (np == 0) {
        if (kout != kin) CUDA_TRY(cudaMemcpyAsync(kout, kin, n * sizeof(K), cudaMemcpyDeviceToDevice, s));
        if (vin && vout != vin)
            CUDA_TRY(cudaMemcpyAsync(vout, vin, n * sizeof(V), cudaMemcpyDeviceToDevice, s));
        return;
    }
    const int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
    // onesweep (default): one global histogram of all passes first, then per pass the
    // single-pass kernel with decoupled look-back.  SLM_SORT_ONESWEEP=0: reduce-then-scan
    // (per pass a tile-histogram kernel, a scan of the digit-major counts, and the same
    // ranking / scatter kernel with known offsets); measured a few % slower.
    static const bool onesweep = !(getenv("SLM_SORT_ONESWEEP") && atoi(getenv("SLM_SORT_ONESWEEP")) == 0);
    unsigned long long *hist = nullptr, *status = nullptr;
    unsigned *tickets = nullptr;
    size_t sb = 0;
    const bool single = ntiles == 1 && onesweep;   // one kernel per pass, nothing else
    if (onesweep && !single) {
        // scratch: [hist np*256 u64 | tickets np u32 (padded) | status ntiles*256 u64]
        const size_t hb = (size_t)np * 256 * 8, tb = 64;
        sb = (size_t)ntiles * 256 * 8;
        ctx->tmp.resize(hb + tb + sb);
        hist = (unsigned long long *)ctx->tmp.p;
        tickets = (unsigned *)((char *)ctx->tmp.p + hb);
        status = (unsigned long long *)((char *)ctx->tmp.p + hb + tb);
        CUDA_TRY(cudaMemsetAsync(ctx->tmp.p, 0, hb + tb, s));
        k_rs_hist<K><<<grid_for(n, 256, SMS() * 8), 256, 0, s>>>(kin, n, begin_bit, np, end_bit,
                                                                 hist);
        k_rs_hist_scan<<<np, 256, 0, s>>>(hist);
    }
    const size_t smem = rs_smem_bytes<K, V>();
    CUDA_TRY(cudaFuncSetAttribute(k_rs_onesweep<K, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    // ping-pong so that the last pass lands in kout / vout
    const K *ks = kin;
    const V *vs = vin;
    DBuf<int32_t> tcnt;
    DBuf<int64_t> toffb;
    if (!onesweep) {
        tcnt.resize(256 * ntiles);
        toffb.resize(256 * ntiles);
    }
    for (int p = 0; p < np; p++) {
        const bool to_out = ((np - 1 - p) % 2) == 0;
        K *kd = to_out ? kout : kalt;
        V *vd = vin ? (to_out ? vout : valt) : nullptr;
        const int shift = begin_bit + 8 * p;
        const unsigned dmask = end_bit - shift >= 8 ? 255u : ((1u << (end_bit - shift)) - 1u);
        const int64_t *toff = nullptr;
        if (single) {
        } else if (onesweep) {
            CUDA_TRY(cudaMemsetAsync(status, 0, sb, s));
        } else {
            k_rs_tilehist<K><<<(unsigned)ntiles, RS_BLOCK, 0, s>>>(ks, n, shift, dmask, ntiles,
                                                                 tcnt.p);
            dev_exclusive_sum<int32_t, int64_t>(ctx, tcnt.p, toffb.p, 256 * ntiles);
            toff = toffb.p;
        }
        k_rs_onesweep<K, V><<<(unsigned)ntiles, RS_BLOCK, smem, s>>>(
            ks, kd, vs, vd, n, shift, dmask, hist ? hist + p * 256 : nullptr, status,
            tickets ? tickets + p : nullptr, toff, ntiles);
        ks = kd;
        vs = vd;
    }
    CUDA_TRY(cudaGetLastError());
}

}  // namespace

// ------------------------------------------------------------------ internal API

template <class TI, class TO>
void dev_exclusive_sum(slm_ctx *ctx, const TI *in, TO *out, int64_t n) {
    scan_run<TI, TO, false>(ctx, in, out, nullptr, n);
}
template void dev_exclusive_sum<int64_t, int64_t>(slm_ctx *, const int64_t *, int64_t *, int64_t);
template void dev_exclusive_sum<int32_t, int32_t>(slm_ctx *, const int32_t *, int32_t *, int64_t);
template void dev_exclusive_sum<int32_t, int64_t>(slm_ctx *, const int32_t *, int64_t *, int64_t);
template void dev_exclusive_sum<double, double>(slm_ctx *, const double *, double *, int64_t);

void dev_exclusive_sum_by_key(slm_ctx *ctx, const uint32_t *keys, const int32_t *in, int32_t *out,
                              int64_t n) {
    scan_run<int32_t, int32_t, true>(ctx, in, out, keys, n);
}

void sort_pairs_u64_f64(slm_ctx *ctx, DBuf<uint64_t> &keys, DBuf<double> &vals, int64_t n,
                        int end_bit) {
    // two buffers, like a double-buffered sort: the caller's arrays (whose input may be
    // overwritten) and the context's u64b / f64b; the result is swapped into keys / vals
    ctx->u64b.resize(n);
    ctx->f64b.resize(n);
    const int np = end_bit > 0 ? (end_bit + 7) / 8 : 0;
    if (np % 2 == 1) {
        // odd pass count: keys -> u64b -> keys ... ends in u64b
        radix_sort_impl<uint64_t, double>(ctx, keys.p, ctx->u64b.p, vals.p, ctx->f64b.p, keys.p,
                                          vals.p, n, 0, end_bit);
        keys.swap(ctx->u64b);
        vals.swap(ctx->f64b);
    } else if (np > 0) {
        // even pass count: keys -> u64b -> keys ... ends in keys
        radix_sort_impl<uint64_t, double>(ctx, keys.p, keys.p, vals.p, vals.p, ctx->u64b.p,
                                          ctx->f64b.p, n, 0, end_bit);
    }
    keys.n = n;
    vals.n = n;
}

void sort_pairs_u32_i32(slm_ctx *ctx, uint32_t *keys_in, uint32_t *keys_out, int32_t *vals_in,
                        int32_t *vals_out, int64_t n, int end_bit) {
    ctx->sort_k32.resize(n);
    ctx->sort_v32.resize(n);
    radix_sort_impl<uint32_t, int32_t>(ctx, keys_in, keys_out, vals_in, vals_out, ctx->sort_k32.p,
                                       ctx->sort_v32.p, n, 0, end_bit);
}

// 32-bit keys with 64-bit payloads (the sweep view's row transposition, slm_build.cu).  A is
// the input and is overwritten; the result lands in B for an odd number of 8-bit passes and
// in A for an even number: returns true when it is in B.
bool sort_pairs_u32_u64(slm_ctx *ctx, uint32_t *kA, uint32_t *kB, uint64_t *vA, uint64_t *vB,
                        int64_t n, int end_bit) {
    const int np = end_bit > 0 ? (end_bit + 7) / 8 : 0;
    if (np == 0) return false;
    if (np % 2 == 1) {
        radix_sort_impl<uint32_t, uint64_t>(ctx, kA, kB, vA, vB, kA, vA, n, 0, end_bit);
        return true;
    }
    radix_sort_impl<uint32_t, uint64_t>(ctx, kA, kA, vA, vA, kB, vB, n, 0, end_bit);
    return false;
}

// diagnostics hooks (slm_capi.cu slm_debug_sort / slm_debug_scan)
double debug_sort(slm_ctx *ctx, int kind, void *keys, void *vals, int64_t n, int end_bit) {
    cudaStream_t s = ctx->stream;
    const size_t kb = kind == 0 ? 8 : 4;
    DBuf<uint8_t> k, v, k2, v2;
    k.resize(n * kb);
    v.resize(n * kb);
    k2.resize(n * kb);
    v2.resize(n * kb);
    CUDA_TRY(cudaMemcpyAsync(k.p, keys, n * kb, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(v.p, vals, n * kb, cudaMemcpyHostToDevice, s));
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventRecord(e0, s));
    if (kind == 0) {
        ctx->sort_k64.resize(n);
        ctx->sort_v64.resize(n);
        radix_sort_impl<uint64_t, double>(ctx, (uint64_t *)k.p, (uint64_t *)k2.p, (double *)v.p,
                                          (double *)v2.p, ctx->sort_k64.p, ctx->sort_v64.p, n, 0,
                                          end_bit);
    } else {
        sort_pairs_u32_i32(ctx, (uint32_t *)k.p, (uint32_t *)k2.p, (int32_t *)v.p, (int32_t *)v2.p,
                           n, end_bit);
    }
    CUDA_TRY(cudaEventRecord(e1, s));
    CUDA_TRY(cudaMemcpyAsync(keys, k2.p, n * kb, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(vals, v2.p, n * kb, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ms;
}

void debug_scan(slm_ctx *ctx, int kind, const void *in, void *out, const uint32_t *keys, int64_t n) {
    cudaStream_t s = ctx->stream;
    const size_t ib = (kind == 1 || kind == 2 || kind == 4) ? 4 : 8;
    const size_t ob = (kind == 1 || kind == 4) ? 4 : 8;
    DBuf<uint8_t> di, dout, dk;
    di.resize(n * ib);
    dout.resize(n * ob);
    CUDA_TRY(cudaMemcpyAsync(di.p, in, n * ib, cudaMemcpyHostToDevice, s));
    if (kind == 4) {
        dk.resize(n * 4);
        CUDA_TRY(cudaMemcpyAsync(dk.p, keys, n * 4, cudaMemcpyHostToDevice, s));
    }
    switch (kind) {
    case 0: dev_exclusive_sum<int64_t, int64_t>(ctx, (int64_t *)di.p, (int64_t *)dout.p, n); break;
    case 1: dev_exclusive_sum<int32_t, int32_t>(ctx, (int32_t *)di.p, (int32_t *)dout.p, n); break;
    case 2: dev_exclusive_sum<int32_t, int64_t>(ctx, (int32_t *)di.p, (int64_t *)dout.p, n); break;
    case 3: dev_exclusive_sum<double, double>(ctx, (double *)di.p, (double *)dout.p, n); break;
    default:
        dev_exclusive_sum_by_key(ctx, (uint32_t *)dk.p, (int32_t *)di.p, (int32_t *)dout.p, n);
    }
    CUDA_TRY(cudaMemcpyAsync(out, dout.p, n * ob, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
}

const void *slm_anchor_prim() { return (const void *)k_rs_hist_scan; }
