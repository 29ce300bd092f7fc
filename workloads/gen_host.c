/* gen_host.c -- host twins of the device graph generators (libslm slm_gen.cu), in plain C.
 *
 * Input generation only: neither product nor oracle.  Both the CPU oracle / reference arm
 * and the tests get their edge lists from here; the product builds the same graphs in HBM
 * with its own device generators (slm_build_rmat / slm_build_rgg), and
 * tests/test_gpu_parity.py checks the two CSRs bit for bit.  Every draw is a pure hash of
 * (seed, edge or point id, stream): SplitMix64's finaliser (the same constants as rng.py:19-23
 * of the reference), so the draws are order-free and the loops below run on every host core.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EXPORT __attribute__((visibility("default")))
#define GAMMA64 0x9E3779B97F4A7C15ULL
#define MIX1 0xBF58476D1CE4E5B9ULL
#define MIX2 0x94D049BB133111EBULL

static inline uint64_t fin(uint64_t z) {
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}
static inline uint64_t base_of(uint64_t seed) { return fin(seed ^ 0x5851F42D4C957F2DULL); }
static inline double unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

/* bijection of [0, 2^scale): three rounds of odd multiply, xor-shift, add */
static inline uint64_t permute(uint64_t x, int scale, uint64_t base) {
    const uint64_t mask = scale >= 64 ? ~0ULL : ((1ULL << scale) - 1);
    const int sh = (scale + 1) / 2;
    for (int r = 0; r < 3; r++) {
        uint64_t k = fin(base + 0x1000ULL + (uint64_t)r);
        x = (x * (k | 1ULL)) & mask;
        x ^= x >> sh;
        x = (x + (k >> 17)) & mask;
    }
    return x;
}

/* R-MAT edge k: one quadrant draw per level against thresholds a, a+b, a+b+c */
static inline void rmat_edge(uint64_t base, int scale, int64_t k, double t1, double t2, double t3,
                             uint64_t *s, uint64_t *d, uint64_t *wh) {
    const uint64_t kb = fin(base + (uint64_t)k * GAMMA64);
    uint64_t a = 0, b = 0;
    for (int l = 0; l < scale; l++) {
        double u = unit(fin(kb + (uint64_t)(l + 1) * MIX1));
        int q = u < t1 ? 0 : (u < t2 ? 1 : (u < t3 ? 2 : 3));
        a = (a << 1) | (uint64_t)(q >> 1);
        b = (b << 1) | (uint64_t)(q & 1);
    }
    *s = permute(a, scale, base);
    *d = permute(b, scale, base);
    *wh = fin(kb + MIX2);
}

#define BLK 65536

/* R-MAT scale / edge_factor, both directions of every non-loop draw; weight 1 or U[1,100].
 * Pass NULL outputs to get the edge count only. */
EXPORT int64_t gen_rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                        int weight_mode, int64_t *src, int64_t *dst, double *w) {
    const uint64_t base = base_of(seed);
    const int64_t m = (int64_t)edge_factor << scale;
    const double t1 = a, t2 = a + b, t3 = a + b + c;
    const int64_t nb = (m + BLK - 1) / BLK;
    int64_t *kept = (int64_t *)calloc((size_t)nb + 1, sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t q = 0; q < nb; q++) {
        int64_t hi = (q + 1) * BLK < m ? (q + 1) * BLK : m, cnt = 0;
        for (int64_t k = q * BLK; k < hi; k++) {
            uint64_t s, d, wh;
            rmat_edge(base, scale, k, t1, t2, t3, &s, &d, &wh);
            cnt += s != d;
        }
        kept[q + 1] = cnt;
    }
    for (int64_t q = 0; q < nb; q++) kept[q + 1] += kept[q];
    const int64_t total = 2 * kept[nb];
    if (src) {
#pragma omp parallel for schedule(dynamic, 4)
        for (int64_t q = 0; q < nb; q++) {
            int64_t hi = (q + 1) * BLK < m ? (q + 1) * BLK : m, p = 2 * kept[q];
            for (int64_t k = q * BLK; k < hi; k++) {
                uint64_t s, d, wh;
                rmat_edge(base, scale, k, t1, t2, t3, &s, &d, &wh);
                if (s == d) continue;
                double x = weight_mode ? (double)(1 + wh % 100ULL) : 1.0;
                src[p] = (int64_t)s; dst[p] = (int64_t)d; w[p] = x;
                src[p + 1] = (int64_t)d; dst[p + 1] = (int64_t)s; w[p + 1] = x;
                p += 2;
            }
        }
    }
    free(kept);
    return total;
}

static inline void rgg_point(uint64_t base, int64_t i, double *x, double *y) {
    uint64_t h1 = fin(base + (uint64_t)i * GAMMA64);
    *x = unit(h1);
    *y = unit(fin(h1 ^ MIX2));
}
static inline int cell_of(double v, int G) {
    int c = (int)(v * G);
    return c >= G ? G - 1 : c;
}

/* Random geometric graph: n uniform points, pairs closer than radius (both directions),
 * unit weights; neighbours found through a G x G grid of cells of side >= radius. */
EXPORT int64_t gen_rgg(int64_t n, double radius, uint64_t seed, int64_t *src, int64_t *dst,
                       double *w) {
    const uint64_t base = base_of(seed);
    int G = (int)floor(1.0 / radius);
    if (G < 1) G = 1;
    const double r2 = radius * radius;
    const int64_t nc = (int64_t)G * G;
    double *X = (double *)malloc((size_t)n * sizeof(double));
    double *Y = (double *)malloc((size_t)n * sizeof(double));
    int64_t *cell = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *cptr = (int64_t *)calloc((size_t)nc + 1, sizeof(int64_t));
    int64_t *pts = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *deg = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        rgg_point(base, i, &X[i], &Y[i]);
        cell[i] = (int64_t)cell_of(Y[i], G) * G + cell_of(X[i], G);
    }
    for (int64_t i = 0; i < n; i++) cptr[cell[i] + 1]++;
    for (int64_t k = 0; k < nc; k++) cptr[k + 1] += cptr[k];
    {
        int64_t *fill = (int64_t *)malloc((size_t)nc * sizeof(int64_t));
        memcpy(fill, cptr, (size_t)nc * sizeof(int64_t));
        for (int64_t i = 0; i < n; i++) pts[fill[cell[i]]++] = i;   /* ascending id per cell */
        free(fill);
    }
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1) {
            if (!src) break;
            for (int64_t i = 0; i < n; i++) deg[i + 1] += deg[i];
        }
#pragma omp parallel for schedule(dynamic, 4096)
        for (int64_t i = 0; i < n; i++) {
            const int cx = (int)(cell[i] % G), cy = (int)(cell[i] / G);
            int64_t k = pass ? deg[i] : 0;
            for (int dy = -1; dy <= 1; dy++)
                for (int dx = -1; dx <= 1; dx++) {
                    const int ux = cx + dx, uy = cy + dy;
                    if (ux < 0 || uy < 0 || ux >= G || uy >= G) continue;
                    const int64_t cc = (int64_t)uy * G + ux;
                    for (int64_t q = cptr[cc]; q < cptr[cc + 1]; q++) {
                        const int64_t j = pts[q];
                        if (j == i) continue;
                        const double ex = X[i] - X[j], ey = Y[i] - Y[j];
                        if (ex * ex + ey * ey < r2) {
                            if (pass) { src[k] = i; dst[k] = j; w[k] = 1.0; }
                            k++;
                        }
                    }
                }
            if (!pass) deg[i + 1] = k;
        }
    }
    int64_t total = 0;
    if (src) total = deg[n];
    else for (int64_t i = 0; i < n; i++) total += deg[i + 1];
    free(X); free(Y); free(cell); free(cptr); free(pts); free(deg);
    return total;
}

/* ---------------------------------------------------------------- pair models
 * Planted-partition SBM and degree-corrected (Chung-Lu) SBM by one Bernoulli draw per node
 * pair i < j: edge iff unit(fin(base + (i * n + j) * GAMMA)) < p_ij, both directions.
 *   mode 0 (SBM):  p_ij = p_in if i / bs == j / bs else p_out  (bs = n / blocks)
 *   mode 1 (DC-SBM): p_ij = min(1, kin_i kin_j / K[c_i]) if c_i == c_j
 *                    else min(1, kout_i kout_j / O)
 * Only IEEE-exact operations (* / < min) touch the per-node parameters, so the device twin
 * (libslm slm_build_pairs) draws the identical edge set. */
static inline double pair_p(int mode, int64_t i, int64_t j, int64_t bs, double p_in, double p_out,
                            const int32_t *comm, const double *kin, const double *kout,
                            const double *K, double O) {
    if (mode == 0) return (i / bs == j / bs) ? p_in : p_out;
    double p = (comm[i] == comm[j]) ? (kin[i] * kin[j]) / K[comm[i]] : (kout[i] * kout[j]) / O;
    return p < 1.0 ? p : 1.0;
}

EXPORT int64_t gen_pairs(int mode, int64_t n, int64_t blocks, double p_in, double p_out,
                         const int32_t *comm, const double *kin, const double *kout,
                         const double *K, double O, uint64_t seed, int64_t *src, int64_t *dst,
                         double *w) {
    const uint64_t base = base_of(seed);
    const int64_t bs = blocks > 0 ? (n / blocks > 0 ? n / blocks : 1) : 1;
    int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1) {
            if (!src) break;
            for (int64_t i = 0; i < n; i++) cnt[i + 1] += cnt[i];
        }
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; i++) {
            int64_t k = pass ? cnt[i] : 0;
            for (int64_t j = i + 1; j < n; j++) {
                const double u = unit(fin(base + (uint64_t)(i * n + j) * GAMMA64));
                if (u < pair_p(mode, i, j, bs, p_in, p_out, comm, kin, kout, K, O)) {
                    if (pass) {
                        src[2 * k] = i; dst[2 * k] = j; w[2 * k] = 1.0;
                        src[2 * k + 1] = j; dst[2 * k + 1] = i; w[2 * k + 1] = 1.0;
                    }
                    k++;
                }
            }
            if (!pass) cnt[i + 1] = k;
        }
    }
    int64_t total = 0;
    if (src) total = 2 * cnt[n];
    else for (int64_t i = 0; i < n; i++) total += 2 * cnt[i + 1];
    free(cnt);
    return total;
}
