/*
 * slm_oracle.c -- CPU restatement of the synclouvain reference (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity oracle for the B200 path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it, and only as the checker
 * (or as the timed CPU baseline); the product library never links or calls it.
 *
 * It restates /root/reference/pkg/src/synclouvain (pure Python + numpy) in plain C, keeping
 * numpy's exact floating-point evaluation orders so that it is bit-identical to the
 * reference even for non-integer weights:
 *   - ndarray.sum()          -> numpy pairwise summation over the (gathered) operand
 *   - np.add.reduceat        -> first element + pairwise(rest of the segment)
 *   - np.bincount(weights=)  -> sequential accumulation in index order starting at 0.0
 *   - every gain expression  -> same operand order, no FMA contraction (-ffp-contract=off)
 * Pinned against the reference itself (tests/test_oracle_vs_reference.py, run where
 * /root/reference exists) and against committed golden vectors (tests/golden/).
 *
 * Node ids are int64 as in the reference (graph.py:87-89); weights fp64.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------ numpy sums */

/* numpy DOUBLE_pairwise_sum (PW_BLOCKSIZE 128, 8-way unroll); used by ndarray.sum(). */
static double pw_sum(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; i++) r += a[i];
        return r;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
    }
}

/* np.add.reduceat segment value: first + pairwise(rest). */
static double reduceat_seg(const double *a, int64_t n) {
    return a[0] + pw_sum(a + 1, n - 1);
}

/* growable double scratch */
typedef struct { double *v; int64_t n, cap; } dvec;
static void dv_clear(dvec *d) { d->n = 0; }
static void dv_push(dvec *d, double x) {
    if (d->n == d->cap) {
        d->cap = d->cap ? d->cap * 2 : 64;
        d->v = (double *)realloc(d->v, (size_t)d->cap * sizeof(double));
    }
    d->v[d->n++] = x;
}
static void dv_free(dvec *d) { free(d->v); d->v = NULL; d->n = d->cap = 0; }

typedef struct { int64_t *v; int64_t n, cap; } ivec;
static void iv_push(ivec *d, int64_t x) {
    if (d->n == d->cap) {
        d->cap = d->cap ? d->cap * 2 : 64;
        d->v = (int64_t *)realloc(d->v, (size_t)d->cap * sizeof(int64_t));
    }
    d->v[d->n++] = x;
}
static void iv_free(ivec *d) { free(d->v); d->v = NULL; d->n = d->cap = 0; }

static int cmp_i64(const void *x, const void *y) {
    int64_t a = *(const int64_t *)x, b = *(const int64_t *)y;
    return (a > b) - (a < b);
}

/* ------------------------------------------------------------- stable argsort */

/* Stable LSD radix argsort of uint64 keys (equivalent to numpy's stable sorts). */
static void radix_argsort_u64(const uint64_t *key, int64_t n, int64_t *perm) {
    uint64_t used = 0;
    for (int64_t i = 0; i < n; i++) { perm[i] = i; used |= key[i]; }
    int64_t *tmp = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t cnt[256];
    for (int shift = 0; shift < 64; shift += 8) {
        if (((used >> shift) & 0xFF) == 0 && (used >> shift) == 0) break;
        if (((used >> shift) & 0xFF) == 0) continue;
        memset(cnt, 0, sizeof(cnt));
        for (int64_t i = 0; i < n; i++) cnt[(key[perm[i]] >> shift) & 0xFF]++;
        int64_t s = 0;
        for (int b = 0; b < 256; b++) { int64_t c = cnt[b]; cnt[b] = s; s += c; }
        for (int64_t i = 0; i < n; i++) tmp[cnt[(key[perm[i]] >> shift) & 0xFF]++] = perm[i];
        memcpy(perm, tmp, (size_t)n * sizeof(int64_t));
    }
    free(tmp);
}

/* ---------------------------------------------------------------- graph core */

typedef struct {
    int64_t n, ne;                     /* nodes, merged directed CSR entries */
    int64_t *out_ptr, *out_dst;        /* graph.py:109-110 */
    double *out_w;
    int64_t ue;                        /* union entries */
    int64_t *uptr, *unbr;              /* graph.py:151-175 (NeighborUnion ptr/nbr) */
    double *uu;                        /* w_out + w_in per union entry (F6) */
    double *s_out, *s_in, m;           /* graph.py:257-263 */
    int64_t *in_ptr, *in_e;            /* in-CSR: CSR entry indices per destination */
    int integral;                      /* every weight an integer, m < 2^52: sums exact */
} orc_graph;

static int g_threads = 1;
EXPORT void orc_set_threads(int t) { g_threads = t > 0 ? t : 1; }

static int cmp_u64(const void *x, const void *y) {
    uint64_t a = *(const uint64_t *)x, b = *(const uint64_t *)y;
    return (a > b) - (a < b);
}
static void sort_u64(uint64_t *v, int64_t n) {
    if (n <= 24) {
        for (int64_t k = 1; k < n; k++) {
            uint64_t x = v[k];
            int64_t q = k - 1;
            while (q >= 0 && v[q] > x) { v[q + 1] = v[q]; q--; }
            v[q + 1] = x;
        }
    } else {
        qsort(v, (size_t)n, sizeof(uint64_t), cmp_u64);
    }
}

/* Bucket entries [0, m) by row[] into a CSR (ptr[n+1], idx[m]) holding, per row, the entry
 * indices in ascending order: the order a stable sort by row produces.  Parallel (atomic
 * counts and fills, then an ascending sort inside each row). */
static void bucket_stable(const int64_t *row, int64_t m, int64_t n, int64_t *ptr, int64_t *idx) {
    memset(ptr, 0, (size_t)(n + 1) * sizeof(int64_t));
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t i = 0; i < m; i++) __atomic_fetch_add(&ptr[row[i] + 1], 1, __ATOMIC_RELAXED);
    for (int64_t r = 0; r < n; r++) ptr[r + 1] += ptr[r];
    int64_t *fill = (int64_t *)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
    memcpy(fill, ptr, (size_t)n * sizeof(int64_t));
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t i = 0; i < m; i++)
        idx[__atomic_fetch_add(&fill[row[i]], 1, __ATOMIC_RELAXED)] = i;
    free(fill);
#pragma omp parallel for schedule(dynamic, 1024) num_threads(g_threads)
    for (int64_t r = 0; r < n; r++)
        sort_u64((uint64_t *)idx + ptr[r], ptr[r + 1] - ptr[r]);
}

/* Union of out- and in-neighbours minus self-loops (graph.py:151-175).  The reference
 * lexsorts the concatenation [forward; reverse] and reduceats each (row, nbr) group; a
 * group holds at most one forward and one reverse entry, so w_out = W(i,j) (+0.0) and
 * w_in = W(j,i) (+0.0) exactly and the consumers' w_out + w_in is W(i,j) + W(j,i).
 * The in-CSR is the stable sort of the CSR entries by destination (graph.py:111-115):
 * per destination, the entries in CSR order, i.e. by ascending source. */
static void build_union(orc_graph *g) {
    int64_t n = g->n, ne = g->ne;
    int64_t *in_ptr = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
    int64_t *in_e = (int64_t *)malloc((size_t)(ne ? ne : 1) * sizeof(int64_t));
    int64_t *esrc = (int64_t *)malloc((size_t)(ne ? ne : 1) * sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 4096) num_threads(g_threads)
    for (int64_t i = 0; i < n; i++)
        for (int64_t e = g->out_ptr[i]; e < g->out_ptr[i + 1]; e++) esrc[e] = i;
    bucket_stable(g->out_dst, ne, n, in_ptr, in_e);
    g->in_ptr = in_ptr;
    g->in_e = in_e;
    g->uptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1) {
            for (int64_t i = 0; i < n; i++) g->uptr[i + 1] += g->uptr[i];
            g->ue = g->uptr[n];
            g->unbr = (int64_t *)malloc((size_t)(g->ue ? g->ue : 1) * sizeof(int64_t));
            g->uu = (double *)malloc((size_t)(g->ue ? g->ue : 1) * sizeof(double));
        }
#pragma omp parallel for schedule(dynamic, 1024) num_threads(g_threads)
        for (int64_t i = 0; i < n; i++) {
            int64_t a = g->out_ptr[i], ae = g->out_ptr[i + 1];
            int64_t b = in_ptr[i], be = in_ptr[i + 1];
            int64_t k = pass ? g->uptr[i] : 0;
            for (;;) {
                while (a < ae && g->out_dst[a] == i) a++;
                while (b < be && esrc[in_e[b]] == i) b++;
                if (a >= ae && b >= be) break;
                int64_t j;
                double u;
                int64_t bs = b < be ? esrc[in_e[b]] : 0;
                if (b >= be || (a < ae && g->out_dst[a] < bs)) {
                    j = g->out_dst[a]; u = g->out_w[a] + 0.0; a++;
                } else if (a >= ae || bs < g->out_dst[a]) {
                    j = bs; u = 0.0 + g->out_w[in_e[b]]; b++;
                } else {
                    j = g->out_dst[a]; u = g->out_w[a] + g->out_w[in_e[b]]; a++; b++;
                }
                if (pass) { g->unbr[k] = j; g->uu[k] = u; }
                k++;
            }
            if (!pass) g->uptr[i + 1] = k;
        }
    }
    free(esrc);
}

/* strengths (graph.py:257-263): bincount (sequential in edge order) for s_out, s_in;
 * pairwise m_w.  s_in[j] accumulates j's in-edges in CSR order = the in-CSR order. */
static void build_strengths(orc_graph *g) {
    int64_t n = g->n;
    g->s_out = (double *)calloc((size_t)(n ? n : 1), sizeof(double));
    g->s_in = (double *)calloc((size_t)(n ? n : 1), sizeof(double));
#pragma omp parallel for schedule(dynamic, 4096) num_threads(g_threads)
    for (int64_t i = 0; i < n; i++) {
        double so = 0.0, si = 0.0;
        for (int64_t e = g->out_ptr[i]; e < g->out_ptr[i + 1]; e++) so += g->out_w[e];
        for (int64_t b = g->in_ptr[i]; b < g->in_ptr[i + 1]; b++) si += g->out_w[g->in_e[b]];
        g->s_out[i] = so;
        g->s_in[i] = si;
    }
    g->m = pw_sum(g->out_w, g->ne);
    int integral = 1;
    for (int64_t e = 0; e < g->ne && integral; e++)
        integral = g->out_w[e] == floor(g->out_w[e]);
    g->integral = integral && g->m < 0x1p52;
}

/* Graph.from_edges (graph.py:84-116): stable lexsort by (src, dst), merge each
 * duplicate run with np.add.reduceat (first + pairwise(rest)), out_ptr by bincount.
 * Done as a stable bucket by src, then per row a sort by (dst, input position): the same
 * order as the stable lexsort, so the runs are merged in the reference's order.
 * Inputs must already be validated by the caller (ValueError path is host-side). */
EXPORT orc_graph *orc_graph_new(int64_t n, const int64_t *src, const int64_t *dst,
                                const double *w, int64_t ne_in) {
    orc_graph *g = (orc_graph *)calloc(1, sizeof(orc_graph));
    g->n = n;
    int64_t *rptr = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
    uint64_t *key = (uint64_t *)malloc((size_t)(ne_in ? ne_in : 1) * sizeof(uint64_t));
    bucket_stable(src, ne_in, n, rptr, (int64_t *)key);
    /* key = dst * 2^31 + position (n, ne_in < 2^31 here: int32 ids) */
    int64_t *gcnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 1024) num_threads(g_threads)
    for (int64_t r = 0; r < n; r++) {
        int64_t lo = rptr[r], hi = rptr[r + 1], c = 0;
        for (int64_t k = lo; k < hi; k++) key[k] = ((uint64_t)dst[key[k]] << 31) | key[k];
        sort_u64(key + lo, hi - lo);
        for (int64_t k = lo; k < hi; k++)
            if (k == lo || (key[k] >> 31) != (key[k - 1] >> 31)) c++;
        gcnt[r + 1] = c;
    }
    for (int64_t r = 0; r < n; r++) gcnt[r + 1] += gcnt[r];
    g->out_ptr = gcnt;
    g->ne = gcnt[n];
    g->out_dst = (int64_t *)malloc((size_t)(g->ne ? g->ne : 1) * sizeof(int64_t));
    g->out_w = (double *)malloc((size_t)(g->ne ? g->ne : 1) * sizeof(double));
#pragma omp parallel num_threads(g_threads)
    {
        dvec seg = {0};
#pragma omp for schedule(dynamic, 1024)
        for (int64_t r = 0; r < n; r++) {
            int64_t lo = rptr[r], hi = rptr[r + 1], o = gcnt[r];
            int64_t k = lo;
            while (k < hi) {
                uint64_t d = key[k] >> 31;
                dv_clear(&seg);
                while (k < hi && (key[k] >> 31) == d) { dv_push(&seg, w[key[k] & 0x7FFFFFFFULL]); k++; }
                g->out_dst[o] = (int64_t)d;
                g->out_w[o] = reduceat_seg(seg.v, seg.n);
                o++;
            }
        }
        dv_free(&seg);
    }
    free(rptr); free(key);
    build_union(g);
    build_strengths(g);
    return g;
}

EXPORT void orc_graph_free(orc_graph *g) {
    if (!g) return;
    free(g->in_ptr); free(g->in_e);
    free(g->out_ptr); free(g->out_dst); free(g->out_w);
    free(g->uptr); free(g->unbr); free(g->uu);
    free(g->s_out); free(g->s_in);
    free(g);
}

EXPORT int orc_graph_integral(const orc_graph *g) { return g->integral; }

EXPORT void orc_graph_sizes(const orc_graph *g, int64_t *n, int64_t *ne, int64_t *ue, double *m) {
    *n = g->n; *ne = g->ne; *ue = g->ue; *m = g->m;
}
EXPORT void orc_graph_csr(const orc_graph *g, int64_t *out_ptr, int64_t *out_dst, double *out_w) {
    memcpy(out_ptr, g->out_ptr, (size_t)(g->n + 1) * sizeof(int64_t));
    memcpy(out_dst, g->out_dst, (size_t)g->ne * sizeof(int64_t));
    memcpy(out_w, g->out_w, (size_t)g->ne * sizeof(double));
}
EXPORT void orc_graph_union(const orc_graph *g, int64_t *uptr, int64_t *unbr, double *uu) {
    memcpy(uptr, g->uptr, (size_t)(g->n + 1) * sizeof(int64_t));
    memcpy(unbr, g->unbr, (size_t)g->ue * sizeof(int64_t));
    memcpy(uu, g->uu, (size_t)g->ue * sizeof(double));
}
/* rows [r0, r1) of the CSR (which = 0) or the union (which = 1), offsets relative to r0;
 * nbr / w nullable (size them from ptr[r1 - r0]) */
EXPORT void orc_graph_rows(const orc_graph *g, int which, int64_t r0, int64_t r1, int64_t *ptr,
                           int64_t *nbr, double *w) {
    const int64_t *P = which ? g->uptr : g->out_ptr;
    const int64_t *N = which ? g->unbr : g->out_dst;
    const double *Wt = which ? g->uu : g->out_w;
    for (int64_t i = 0; i <= r1 - r0; i++) ptr[i] = P[r0 + i] - P[r0];
    int64_t cnt = P[r1] - P[r0];
    if (nbr) memcpy(nbr, N + P[r0], (size_t)cnt * sizeof(int64_t));
    if (w) memcpy(w, Wt + P[r0], (size_t)cnt * sizeof(double));
}
EXPORT void orc_graph_strengths(const orc_graph *g, double *s_out, double *s_in) {
    memcpy(s_out, g->s_out, (size_t)g->n * sizeof(double));
    memcpy(s_in, g->s_in, (size_t)g->n * sizeof(double));
}

/* aggregate (graph.py:266-280): labels must be dense 0..c-1 (checked by the caller). */
EXPORT orc_graph *orc_aggregate(const orc_graph *g, const int64_t *labels, int64_t c) {
    int64_t ne = g->ne;
    int64_t *s = (int64_t *)malloc((size_t)(ne ? ne : 1) * sizeof(int64_t));
    int64_t *d = (int64_t *)malloc((size_t)(ne ? ne : 1) * sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 4096) num_threads(g_threads)
    for (int64_t i = 0; i < g->n; i++)
        for (int64_t e = g->out_ptr[i]; e < g->out_ptr[i + 1]; e++) {
            s[e] = labels[i];
            d[e] = labels[g->out_dst[e]];
        }
    orc_graph *h = orc_graph_new(c, s, d, g->out_w, ne);
    free(s); free(d);
    return h;
}

/* ------------------------------------------------------------------ ASSIGN */

/* _assign_targets / find_assignment (detector.py:123-158): per row the first
 * neighbour (lowest id) maximising the pairwise merge gain; self unless max > 0. */
EXPORT void orc_assign(const orc_graph *g, double m, int64_t *a) {
    const double m2 = m * m;
    const int64_t n = g->n;
#pragma omp parallel for schedule(dynamic, 1024) num_threads(g_threads)
    for (int64_t r = 0; r < n; r++) {
        int64_t e0 = g->uptr[r], e1 = g->uptr[r + 1];
        a[r] = r;
        if (e1 == e0) continue;
        double so = g->s_out[r], si = g->s_in[r];
        double mx = -INFINITY;
        int64_t first = -1;
        for (int64_t e = e0; e < e1; e++) {
            int64_t j = g->unbr[e];
            double gv = g->uu[e] / m - (so * g->s_in[j] + si * g->s_out[j]) / m2;
            if (first < 0 || gv > mx) { mx = gv; first = e; }
        }
        if (mx > 0.0) a[r] = g->unbr[first];
    }
}

/* ------------------------------------------------------------- COMPONENTS */

/* extract_components (forest.py:43-67) + canonicalize_labels (graph.py:283-291): WCC of
 * i -> a[i], labels ordered by smallest member, on_cycle flags.  Returns n_comms. */
EXPORT int64_t orc_components(int64_t n, const int64_t *a, int64_t *comm, uint8_t *on_cycle) {
    if (n == 0) return 0;
    uint8_t *state = (uint8_t *)calloc((size_t)n, 1);
    int64_t *key = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *path = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    memset(on_cycle, 0, (size_t)n);
    for (int64_t s = 0; s < n; s++) {
        if (state[s]) continue;
        int64_t len = 0, x = s;
        while (state[x] == 0) { state[x] = 1; path[len++] = x; x = a[x]; }
        int64_t k;
        if (state[x] == 1) {               /* fresh cycle entered at x */
            int64_t p0 = 0;
            while (path[p0] != x) p0++;
            int64_t mn = x;
            for (int64_t p = p0; p < len; p++) { on_cycle[path[p]] = 1; if (path[p] < mn) mn = path[p]; }
            k = mn;
        } else {
            k = key[x];
        }
        for (int64_t p = 0; p < len; p++) { key[path[p]] = k; state[path[p]] = 2; }
    }
    int64_t *lab = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) lab[i] = -1;
    int64_t next = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t k = key[i];
        if (lab[k] < 0) lab[k] = next++;
        comm[i] = lab[k];
    }
    free(state); free(key); free(path); free(lab);
    return next;
}

/* ------------------------------------------------------------- AGGREGATES */

/* CommunityAggregates.from_labels (quality.py:71-79): sequential bincount. */
static void aggregates(const orc_graph *g, const int64_t *lab, int64_t nc,
                       double *S_out, double *S_in, int64_t *cnt) {
    memset(S_out, 0, (size_t)nc * sizeof(double));
    memset(S_in, 0, (size_t)nc * sizeof(double));
    memset(cnt, 0, (size_t)nc * sizeof(int64_t));
    for (int64_t i = 0; i < g->n; i++) {
        S_out[lab[i]] += g->s_out[i];
        S_in[lab[i]] += g->s_in[i];
        cnt[lab[i]]++;
    }
}

EXPORT void orc_aggregates(const orc_graph *g, const int64_t *lab, int64_t nc,
                           double *S_out, double *S_in, int64_t *cnt) {
    aggregates(g, lab, nc, S_out, S_in, cnt);
}

/* local_gains (quality.py:170-183). */
EXPORT void orc_local_gains(const orc_graph *g, double m, const int64_t *lab, int64_t nc, double *lg) {
    int64_t n = g->n;
    if (m == 0.0) { memset(lg, 0, (size_t)n * sizeof(double)); return; }
    double *S_out = (double *)malloc((size_t)(nc ? nc : 1) * sizeof(double));
    double *S_in = (double *)malloc((size_t)(nc ? nc : 1) * sizeof(double));
    int64_t *cnt = (int64_t *)malloc((size_t)(nc ? nc : 1) * sizeof(int64_t));
    aggregates(g, lab, nc, S_out, S_in, cnt);
#pragma omp parallel for schedule(dynamic, 4096) num_threads(g_threads)
    for (int64_t i = 0; i < n; i++) {
        double w_own = 0.0;
        for (int64_t e = g->uptr[i]; e < g->uptr[i + 1]; e++)
            if (lab[g->unbr[e]] == lab[i]) w_own += g->uu[e];
        int64_t c = lab[i];
        double so = g->s_out[i], si = g->s_in[i];
        lg[i] = w_own / m - (so * (S_in[c] - si) + si * (S_out[c] - so)) / (m * m);
    }
    free(S_out); free(S_in); free(cnt);
}

/* --------------------------------------------------------------- POSITIVE */

typedef struct {
    const orc_graph *g;
    double m, m2;
    int64_t *a;
    int64_t scc_cap;
    /* scratch, sized n */
    int64_t *stamp;       /* membership stamp of the current part */
    int64_t cur;          /* current stamp */
    uint8_t *in_b;
    int64_t *posof;       /* index of node inside current part */
    dvec ws, tmp;
    /* outputs */
    dvec gains;
    int64_t unresolved, n_warn;
    int changed;
} pos_ctx;

static inline int in_mem(const pos_ctx *P, int64_t x) { return P->stamp[x] == P->cur; }

/* _detach_gain (detector.py:178-194) for sorted b_nodes (in_b already marked). */
static double detach_gain(pos_ctx *P, const int64_t *b, int64_t nb, double so_c, double si_c) {
    const orc_graph *g = P->g;
    double x_w = 0.0;
    for (int64_t k = 0; k < nb; k++) {
        int64_t y = b[k];
        int any = 0;
        dv_clear(&P->ws);
        for (int64_t e = g->uptr[y]; e < g->uptr[y + 1]; e++) {
            int64_t z = g->unbr[e];
            if (!in_mem(P, z)) continue;
            any = 1;
            if (!P->in_b[z]) dv_push(&P->ws, g->uu[e]);
        }
        if (any) x_w += pw_sum(P->ws.v, P->ws.n);
    }
    dv_clear(&P->tmp);
    for (int64_t k = 0; k < nb; k++) dv_push(&P->tmp, g->s_out[b[k]]);
    double so_b = pw_sum(P->tmp.v, P->tmp.n);
    dv_clear(&P->tmp);
    for (int64_t k = 0; k < nb; k++) dv_push(&P->tmp, g->s_in[b[k]]);
    double si_b = pw_sum(P->tmp.v, P->tmp.n);
    double null = (-so_c * si_b - so_b * si_c) + 2.0 * so_b * si_b;
    return -x_w / P->m - null / (P->m * P->m);
}

/* _find_cycle (detector.py:163-175): cycle reached from start, rotated to min first. */
static int64_t find_cycle(const int64_t *a, int64_t start, ivec *cyc, int64_t *seen_pos,
                          ivec *path) {
    path->n = 0;
    int64_t x = start;
    while (seen_pos[x] < 0) {
        seen_pos[x] = path->n;
        iv_push(path, x);
        x = a[x];
    }
    int64_t p0 = seen_pos[x];
    int64_t s = path->n - p0;
    int64_t kmin = p0;
    for (int64_t p = p0; p < path->n; p++) if (path->v[p] < path->v[kmin]) kmin = p;
    cyc->n = 0;
    for (int64_t q = 0; q < s; q++) iv_push(cyc, path->v[p0 + (kmin - p0 + q) % s]);
    for (int64_t p = 0; p < path->n; p++) seen_pos[path->v[p]] = -1;
    return s;
}

/* _split_community (detector.py:197-285) on one bad community (members ascending). */
static void split_community(pos_ctx *P, const int64_t *members, int64_t nmem, int64_t *seen_pos) {
    const orc_graph *g = P->g;
    const double m = P->m, m2 = P->m2;
    int64_t *a = P->a;
    /* stack of parts; each part is a sorted malloc'd array */
    typedef struct { int64_t *v; int64_t n; } part_t;
    part_t *stack = NULL;
    int64_t sn = 0, scap = 0;
#define PUSH(ptr, cnt) do { if (sn == scap) { scap = scap ? 2 * scap : 16; \
        stack = (part_t *)realloc(stack, (size_t)scap * sizeof(part_t)); } \
        stack[sn].v = (ptr); stack[sn].n = (cnt); sn++; } while (0)
    int64_t *first = (int64_t *)malloc((size_t)nmem * sizeof(int64_t));
    memcpy(first, members, (size_t)nmem * sizeof(int64_t));
    qsort(first, (size_t)nmem, sizeof(int64_t), cmp_i64);
    PUSH(first, nmem);
    ivec cyc = {0}, path = {0}, sub = {0};
    double *gv = NULL; int64_t gcap = 0;
    int64_t *ch_ptr = NULL, *ch_list = NULL; int64_t chcap = 0;
    uint8_t *is_cyc = NULL;
    while (sn > 0) {
        part_t pt = stack[--sn];
        int64_t *mem = pt.v, pn = pt.n;
        if (pn <= 1) { free(mem); continue; }
        P->cur++;
        for (int64_t k = 0; k < pn; k++) { P->stamp[mem[k]] = P->cur; P->posof[mem[k]] = k; }
        dv_clear(&P->tmp);
        for (int64_t k = 0; k < pn; k++) dv_push(&P->tmp, g->s_out[mem[k]]);
        double so_c = pw_sum(P->tmp.v, P->tmp.n);
        dv_clear(&P->tmp);
        for (int64_t k = 0; k < pn; k++) dv_push(&P->tmp, g->s_in[mem[k]]);
        double si_c = pw_sum(P->tmp.v, P->tmp.n);
        if (gcap < pn) { gcap = pn; gv = (double *)realloc(gv, (size_t)gcap * sizeof(double)); }
        int any_neg = 0;
        for (int64_t k = 0; k < pn; k++) {
            int64_t x = mem[k];
            dv_clear(&P->ws);
            for (int64_t e = g->uptr[x]; e < g->uptr[x + 1]; e++)
                if (in_mem(P, g->unbr[e])) dv_push(&P->ws, g->uu[e]);
            double w_in_c = pw_sum(P->ws.v, P->ws.n);
            gv[k] = w_in_c / m - (g->s_out[x] * (si_c - g->s_in[x]) + g->s_in[x] * (so_c - g->s_out[x])) / m2;
            if (gv[k] < 0.0) any_neg = 1;
        }
        if (!any_neg) { free(mem); continue; }
        int64_t s = find_cycle(a, mem[0], &cyc, seen_pos, &path);
        /* children restricted to the part, ascending (detector.py:229-233) */
        if (chcap < pn) {
            chcap = pn;
            ch_ptr = (int64_t *)realloc(ch_ptr, (size_t)(chcap + 1) * sizeof(int64_t));
            ch_list = (int64_t *)realloc(ch_list, (size_t)chcap * sizeof(int64_t));
            is_cyc = (uint8_t *)realloc(is_cyc, (size_t)chcap);
        }
        memset(ch_ptr, 0, (size_t)(pn + 1) * sizeof(int64_t));
        memset(is_cyc, 0, (size_t)pn);
        for (int64_t q = 0; q < s; q++) is_cyc[P->posof[cyc.v[q]]] = 1;
        for (int64_t k = 0; k < pn; k++) {
            int64_t t = a[mem[k]];
            if (t != mem[k] && in_mem(P, t)) ch_ptr[P->posof[t] + 1]++;
        }
        for (int64_t k = 0; k < pn; k++) ch_ptr[k + 1] += ch_ptr[k];
        {
            int64_t *fill = (int64_t *)malloc((size_t)pn * sizeof(int64_t));
            memcpy(fill, ch_ptr, (size_t)pn * sizeof(int64_t));
            for (int64_t k = 0; k < pn; k++) {
                int64_t t = a[mem[k]];
                if (t != mem[k] && in_mem(P, t)) ch_list[fill[P->posof[t]]++] = mem[k];
            }
            free(fill);
        }
        double best_gain = 0.0;
        int64_t *best_parts = NULL, best_n = 0;
        int64_t cut0 = -1, cut1 = -1;
        /* branch cuts (detector.py:238-253) */
        for (int64_t k = 0; k < pn; k++) {
            if (is_cyc[k]) continue;
            int64_t x = mem[k];
            sub.n = 0;
            iv_push(&sub, x);
            for (int64_t qi = 0; qi < sub.n; qi++) {
                int64_t y = sub.v[qi], py = P->posof[y];
                for (int64_t c = ch_ptr[py]; c < ch_ptr[py + 1]; c++) iv_push(&sub, ch_list[c]);
            }
            qsort(sub.v, (size_t)sub.n, sizeof(int64_t), cmp_i64);
            for (int64_t q = 0; q < sub.n; q++) P->in_b[sub.v[q]] = 1;
            double gsp = detach_gain(P, sub.v, sub.n, so_c, si_c);
            for (int64_t q = 0; q < sub.n; q++) P->in_b[sub.v[q]] = 0;
            if (gsp > best_gain) {
                best_gain = gsp;
                free(best_parts);
                best_parts = (int64_t *)malloc((size_t)sub.n * sizeof(int64_t));
                memcpy(best_parts, sub.v, (size_t)sub.n * sizeof(int64_t));
                best_n = sub.n;
                cut0 = x; cut1 = -1;
            }
        }
        if (best_parts == NULL && s >= 2) {
            if (s > P->scc_cap) {
                /* peel the worst negative cycle node (detector.py:255-268) */
                int64_t worst = -1; double wg = 0.0;
                for (int64_t q = 0; q < s; q++) {
                    int64_t x = cyc.v[q];
                    double gx = gv[P->posof[x]];
                    if (gx < 0.0 && (worst < 0 || gx < wg || (gx == wg && x < worst))) { worst = x; wg = gx; }
                }
                if (worst >= 0) {
                    a[worst] = worst;
                    P->changed = 1;
                    P->n_warn++;
                    PUSH(mem, pn);
                    continue;
                }
            } else {
                /* _best_pair_cut (detector.py:288-335) */
                int64_t **grp = (int64_t **)malloc((size_t)s * sizeof(int64_t *));
                int64_t *gn = (int64_t *)malloc((size_t)s * sizeof(int64_t));
                double *so_g = (double *)malloc((size_t)s * sizeof(double));
                double *si_g = (double *)malloc((size_t)s * sizeof(double));
                for (int64_t q = 0; q < s; q++) {
                    sub.n = 0;
                    iv_push(&sub, cyc.v[q]);
                    for (int64_t qi = 0; qi < sub.n; qi++) {
                        int64_t py = P->posof[sub.v[qi]];
                        for (int64_t c = ch_ptr[py]; c < ch_ptr[py + 1]; c++)
                            if (!is_cyc[P->posof[ch_list[c]]]) iv_push(&sub, ch_list[c]);
                    }
                    qsort(sub.v, (size_t)sub.n, sizeof(int64_t), cmp_i64);
                    grp[q] = (int64_t *)malloc((size_t)sub.n * sizeof(int64_t));
                    memcpy(grp[q], sub.v, (size_t)sub.n * sizeof(int64_t));
                    gn[q] = sub.n;
                    dv_clear(&P->tmp);
                    for (int64_t k = 0; k < sub.n; k++) dv_push(&P->tmp, g->s_out[sub.v[k]]);
                    so_g[q] = pw_sum(P->tmp.v, P->tmp.n);
                    dv_clear(&P->tmp);
                    for (int64_t k = 0; k < sub.n; k++) dv_push(&P->tmp, g->s_in[sub.v[k]]);
                    si_g[q] = pw_sum(P->tmp.v, P->tmp.n);
                }
                double pbest = 0.0;
                int64_t bp = -1, bq = -1;
                dvec wsi = {0};
                for (int64_t p = 0; p < s - 1; p++) {
                    for (int64_t k = 0; k < pn; k++) P->in_b[mem[k]] = 0; /* in_b[:] = False */
                    double so_b = 0.0, si_b = 0.0, x_w = 0.0;
                    for (int64_t q = p + 1; q < s; q++) {
                        for (int64_t k = 0; k < gn[q]; k++) {
                            int64_t y = grp[q][k];
                            int any = 0;
                            dv_clear(&P->ws); dv_clear(&wsi);
                            for (int64_t e = g->uptr[y]; e < g->uptr[y + 1]; e++) {
                                int64_t z = g->unbr[e];
                                if (!in_mem(P, z)) continue;
                                any = 1;
                                if (P->in_b[z]) dv_push(&wsi, g->uu[e]);
                                else dv_push(&P->ws, g->uu[e]);
                            }
                            if (any) x_w += pw_sum(P->ws.v, P->ws.n) - pw_sum(wsi.v, wsi.n);
                            P->in_b[y] = 1;
                        }
                        so_b += so_g[q];
                        si_b += si_g[q];
                        double null = (-so_c * si_b - so_b * si_c) + 2.0 * so_b * si_b;
                        double gain = -x_w / m - null / m2;
                        if (gain > pbest) { pbest = gain; bp = p; bq = q; }
                    }
                }
                for (int64_t k = 0; k < pn; k++) P->in_b[mem[k]] = 0;
                dv_free(&wsi);
                if (bp >= 0 && pbest > best_gain) {
                    best_gain = pbest;
                    int64_t tot = 0;
                    for (int64_t q = bp + 1; q <= bq; q++) tot += gn[q];
                    best_parts = (int64_t *)malloc((size_t)tot * sizeof(int64_t));
                    best_n = 0;
                    for (int64_t q = bp + 1; q <= bq; q++)
                        for (int64_t k = 0; k < gn[q]; k++) best_parts[best_n++] = grp[q][k];
                    qsort(best_parts, (size_t)best_n, sizeof(int64_t), cmp_i64);
                    cut0 = cyc.v[bp]; cut1 = cyc.v[bq];
                }
                for (int64_t q = 0; q < s; q++) free(grp[q]);
                free(grp); free(gn); free(so_g); free(si_g);
            }
        }
        if (best_parts == NULL) {
            for (int64_t k = 0; k < pn; k++) if (gv[k] < 0.0) P->unresolved++;
            free(mem);
            continue;
        }
        a[cut0] = cut0;
        if (cut1 >= 0) a[cut1] = cut1;
        P->changed = 1;
        dv_push(&P->gains, best_gain);
        /* rest = mem minus best_parts (both sorted) */
        int64_t *rest = (int64_t *)malloc((size_t)pn * sizeof(int64_t));
        int64_t rn = 0, bi = 0;
        for (int64_t k = 0; k < pn; k++) {
            while (bi < best_n && best_parts[bi] < mem[k]) bi++;
            if (bi < best_n && best_parts[bi] == mem[k]) continue;
            rest[rn++] = mem[k];
        }
        free(mem);
        PUSH(rest, rn);
        PUSH(best_parts, best_n);
    }
#undef PUSH
    free(stack); free(gv); free(ch_ptr); free(ch_list); free(is_cyc);
    iv_free(&cyc); iv_free(&path); iv_free(&sub);
}

/* positive_correction (detector.py:338-362).  a is updated in place; returns changed.
 * gains_out (nullable) receives up to gains_cap gains in the reference's order. */
EXPORT int orc_positive(const orc_graph *g, double m, int64_t *a, const int64_t *comm,
                        int64_t nc, int64_t scc_cap, int64_t *splits, int64_t *unresolved,
                        double *gains_out, int64_t gains_cap, int64_t *n_warn) {
    int64_t n = g->n;
    double *lg = (double *)malloc((size_t)(n ? n : 1) * sizeof(double));
    orc_local_gains(g, m, comm, nc, lg);
    uint8_t *bad = (uint8_t *)calloc((size_t)(nc ? nc : 1), 1);
    int64_t nbad = 0;
    for (int64_t i = 0; i < n; i++) if (lg[i] < 0.0 && !bad[comm[i]]) { bad[comm[i]] = 1; nbad++; }
    free(lg);
    *splits = 0; *unresolved = 0; *n_warn = 0;
    if (nbad == 0) { free(bad); return 0; }
    /* community_members (forest.py:33-40): ascending ids per community */
    int64_t *cptr = (int64_t *)calloc((size_t)nc + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) cptr[comm[i] + 1]++;
    for (int64_t c = 0; c < nc; c++) cptr[c + 1] += cptr[c];
    int64_t *cmem = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *fill = (int64_t *)malloc((size_t)(nc ? nc : 1) * sizeof(int64_t));
    memcpy(fill, cptr, (size_t)nc * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) cmem[fill[comm[i]]++] = i;
    free(fill);
    pos_ctx P;
    memset(&P, 0, sizeof(P));
    P.g = g; P.m = m; P.m2 = m * m; P.a = a; P.scc_cap = scc_cap;
    P.stamp = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    P.in_b = (uint8_t *)calloc((size_t)n, 1);
    P.posof = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *seen_pos = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) seen_pos[i] = -1;
    for (int64_t c = 0; c < nc; c++) {
        if (!bad[c]) continue;
        split_community(&P, cmem + cptr[c], cptr[c + 1] - cptr[c], seen_pos);
    }
    *splits = P.gains.n;
    *unresolved = P.unresolved;
    *n_warn = P.n_warn;
    if (gains_out) {
        int64_t k = P.gains.n < gains_cap ? P.gains.n : gains_cap;
        memcpy(gains_out, P.gains.v, (size_t)k * sizeof(double));
    }
    int changed = P.changed;
    free(P.stamp); free(P.in_b); free(P.posof); free(seen_pos);
    dv_free(&P.ws); dv_free(&P.tmp); dv_free(&P.gains);
    free(cptr); free(cmem); free(bad);
    return changed;
}

/* ------------------------------------------------- POSITIVE, exact-sum fast form */
/*
 * orc_positive_fast: the same function as orc_positive (detector.py:197-362) for graphs
 * whose weights are integers with m < 2^52 (orc_graph_integral), where every sum the
 * reference forms -- w_in_c, so_c, si_c, x_w, so_b, si_b -- is an exact integer in fp64
 * whatever the summation order.  Only the ORDER of evaluation is changed; every gain is
 * then computed with the reference's fp64 expression on identical operands, so the cuts,
 * the gains list and the unresolved counts are bit-identical.  Cross-checked against the
 * literal restatement above on every integer-weight golden graph and on random graphs
 * (tests/test_oracle.py::test_positive_fast_matches_literal).
 *
 * Per community, over the assignment tree (cycle nodes = roots, depth 0):
 *   W[y]  = weight from y to the members of y's current part      (w_in_c of y)
 *   D[v]  = weight of the part's internal edges whose tree LCA is v
 *   SW, SD, SO, SI = subtree sums of W, D, s_out, s_in
 * so that for the branch cut at x (detector.py:238-253): b = subtree(x),
 *   x_w(b) = SW[x] - 2 SD[x],  so_b = SO[x],  si_b = SI[x]
 * and for the 2-cycle pair cut (detector.py:288-335 with s = 2): b = tree of cyc[1],
 *   x_w = SW[cyc[1]] - 2 SD[cyc[1]] (cross-tree edges have no LCA).  A cut moves b out of
 * the part: ancestors of the cut lose b's sums, every cross edge (y in b, z in rest)
 * lowers W[y], W[z] (and their ancestors' SW) and drops its deposit.  Each part
 * evaluation is then one O(part) scan instead of a breadth-first search per member.
 * Communities whose cycle is longer than 2 (never produced by run()) are
 * handed to the literal form.
 */
typedef struct {
    const orc_graph *g;
    double m, m2;
    int64_t *a;
    int64_t *part;            /* current part id per node (globally unique ids) */
    int64_t *depth;
    uint8_t *root, *cycf;     /* part root (cycle node or cut node); on the part's cycle */
    double *W, *D, *SW, *SD, *SO, *SI;
    int64_t *pos;             /* position of a node inside its community's member list */
} pf_ctx;

static int64_t g_part_next = 1;
static inline int64_t pf_new_part(void) { return __atomic_fetch_add(&g_part_next, 1, __ATOMIC_RELAXED); }
static inline int64_t pf_part(const pf_ctx *F, int64_t z) { return __atomic_load_n(&F->part[z], __ATOMIC_RELAXED); }

static int64_t pf_lca(const pf_ctx *F, int64_t y, int64_t z) {
    const int64_t *a = F->a, *dp = F->depth;
    while (dp[y] > dp[z]) y = a[y];
    while (dp[z] > dp[y]) z = a[z];
    while (y != z) {
        if (F->root[y] || F->root[z]) return -1;
        y = a[y];
        z = a[z];
    }
    return y;
}
/* add dx to SW (which = 0) or SD (which = 1) from v up to its part root */
static void pf_up(pf_ctx *F, int64_t v, double dx, int which) {
    double *S = which ? F->SD : F->SW;
    for (;;) {
        S[v] += dx;
        if (F->root[v]) break;
        v = F->a[v];
    }
}

typedef struct { int64_t *v; int64_t n; int64_t pid; } pf_part_t;

/* one community; returns 0, or -1 when it must go to the literal form (cycle > 2) */
static int pf_split(pf_ctx *F, const int64_t *members, int64_t nmem, dvec *gains_out,
                    int64_t *unresolved_out, int *changed_out, int par) {
    const orc_graph *g = F->g;
    const double m = F->m, m2 = F->m2;
    int64_t *a = F->a;
    /* cycle of the community (from its smallest member, like _find_cycle) */
    int64_t c0 = -1, c1 = -1;
    {
        int64_t x = members[0];
        for (int64_t k = 0; k <= nmem + 1; k++) x = a[x];   /* now on the cycle */
        int64_t y = a[x], len = 1, mn = x;
        while (y != x) { if (y < mn) mn = y; y = a[y]; len++; if (len > 2) return -1; }
        c0 = mn;
        c1 = (len == 2) ? a[mn] : -1;
    }
    const int64_t pid0 = pf_new_part();
    for (int64_t k = 0; k < nmem; k++) {
        int64_t x = members[k];
        F->pos[x] = k;
        __atomic_store_n(&F->part[x], pid0, __ATOMIC_RELAXED);
        F->root[x] = (x == c0 || x == c1);
        F->cycf[x] = F->root[x];
    }
    /* children (non-cycle nodes under their target), community-local CSR by position */
    int64_t *kids = NULL;
    int64_t *cp = (int64_t *)calloc((size_t)nmem + 1, sizeof(int64_t));
    for (int64_t k = 0; k < nmem; k++) {
        int64_t x = members[k];
        if (!F->cycf[x]) cp[F->pos[a[x]] + 1]++;
    }
    for (int64_t k = 0; k < nmem; k++) cp[k + 1] += cp[k];
    kids = (int64_t *)malloc((size_t)(cp[nmem] ? cp[nmem] : 1) * sizeof(int64_t));
    {
        int64_t *fill = (int64_t *)malloc((size_t)(nmem ? nmem : 1) * sizeof(int64_t));
        memcpy(fill, cp, (size_t)nmem * sizeof(int64_t));
        for (int64_t k = 0; k < nmem; k++) {
            int64_t x = members[k];
            if (!F->cycf[x]) kids[fill[F->pos[a[x]]]++] = x;
        }
        free(fill);
    }
    /* depth-ordered layout (BFS from the roots): depths, then bottom-up subtree sums */
    int64_t *bfs = (int64_t *)malloc((size_t)nmem * sizeof(int64_t));
    int64_t nb = 0;
    bfs[nb++] = c0;
    F->depth[c0] = 0;
    if (c1 >= 0) { bfs[nb++] = c1; F->depth[c1] = 0; }
    for (int64_t q = 0; q < nb; q++) {
        int64_t v = bfs[q];
        for (int64_t c = cp[F->pos[v]]; c < cp[F->pos[v] + 1]; c++) {
            F->depth[kids[c]] = F->depth[v] + 1;
            bfs[nb++] = kids[c];
        }
    }
    /* W and the LCA deposits */
    for (int64_t k = 0; k < nmem; k++) {
        int64_t x = members[k];
        double wsum = 0.0;
        for (int64_t e = g->uptr[x]; e < g->uptr[x + 1]; e++) {
            int64_t z = g->unbr[e];
            if (pf_part(F, z) != pid0) continue;
            wsum += g->uu[e];
        }
        F->W[x] = wsum;
        F->D[x] = 0.0;
    }
    for (int64_t k = 0; k < nmem; k++) {
        int64_t x = members[k];
        for (int64_t e = g->uptr[x]; e < g->uptr[x + 1]; e++) {
            int64_t z = g->unbr[e];
            if (z <= x || pf_part(F, z) != pid0) continue;
            int64_t l = pf_lca(F, x, z);
            if (l >= 0) F->D[l] += g->uu[e];
        }
    }
    for (int64_t k = 0; k < nmem; k++) {
        int64_t x = members[k];
        F->SW[x] = F->W[x]; F->SD[x] = F->D[x];
        F->SO[x] = g->s_out[x]; F->SI[x] = g->s_in[x];
    }
    for (int64_t q = nb - 1; q >= 0; q--) {
        int64_t x = bfs[q];
        if (F->cycf[x]) continue;
        int64_t p = a[x];
        F->SW[p] += F->SW[x]; F->SD[p] += F->SD[x];
        F->SO[p] += F->SO[x]; F->SI[p] += F->SI[x];
    }
    free(bfs);
    /* LIFO stack of parts (detector.py:208-284) */
    pf_part_t *stack = (pf_part_t *)malloc(16 * sizeof(pf_part_t));
    int64_t sn = 0, scap = 16;
    {
        int64_t *first = (int64_t *)malloc((size_t)nmem * sizeof(int64_t));
        memcpy(first, members, (size_t)nmem * sizeof(int64_t));
        stack[sn++] = (pf_part_t){first, nmem, pid0};
    }
    int64_t *sub = (int64_t *)malloc((size_t)nmem * sizeof(int64_t));
    while (sn > 0) {
        pf_part_t pt = stack[--sn];
        int64_t *mem = pt.v, pn = pt.n, pid = pt.pid;
        if (pn <= 1) { free(mem); continue; }
        /* roots of this part: its cycle */
        int64_t r0 = -1, r1 = -1;
        {
            int64_t x = mem[0];
            while (!F->root[x]) x = a[x];
            if (a[x] == x) r0 = x;
            else { r0 = x < a[x] ? x : a[x]; r1 = x < a[x] ? a[x] : x; }
        }
        const double so_c = F->SO[r0] + (r1 >= 0 ? F->SO[r1] : 0.0);
        const double si_c = F->SI[r0] + (r1 >= 0 ? F->SI[r1] : 0.0);
        int64_t nneg = 0;
        double best_gain = 0.0;
        int64_t best_x = -1;
#pragma omp parallel num_threads(g_threads) if (par && pn > 65536)
        {
            int64_t my_neg = 0, my_x = -1;
            double my_best = 0.0;
#pragma omp for schedule(static) nowait
            for (int64_t k = 0; k < pn; k++) {
                int64_t x = mem[k];
                double so = g->s_out[x], si = g->s_in[x];
                double gx = F->W[x] / m - (so * (si_c - si) + si * (so_c - so)) / m2;
                if (gx < 0.0) my_neg++;
                if (x == r0 || x == r1) continue;
                double x_w = F->SW[x] - 2.0 * F->SD[x];
                double so_b = F->SO[x], si_b = F->SI[x];
                double null = (-so_c * si_b - so_b * si_c) + 2.0 * so_b * si_b;
                double gsp = -x_w / m - null / (m * m);
                if (gsp > my_best) { my_best = gsp; my_x = x; }   /* first max in this chunk */
            }
#pragma omp critical
            {
                nneg += my_neg;
                if (my_x >= 0 && (my_best > best_gain || (my_best == best_gain && best_x >= 0 && my_x < best_x))) {
                    best_gain = my_best;
                    best_x = my_x;
                }
            }
        }
        if (nneg == 0) { free(mem); continue; }
        int pair = 0;
        if (best_x < 0 && r1 >= 0) {
            /* pair cut of the 2-cycle: b = tree of the larger cycle node */
            double x_w = F->SW[r1] - 2.0 * F->SD[r1];
            double so_b = F->SO[r1], si_b = F->SI[r1];
            double null = (-so_c * si_b - so_b * si_c) + 2.0 * so_b * si_b;
            double gain = -x_w / m - null / m2;
            if (gain > 0.0) { best_gain = gain; best_x = r1; pair = 1; }
        }
        if (best_x < 0) { *unresolved_out += nneg; free(mem); continue; }
        /* apply the cut: b = subtree(best_x) (tree of r1 for the pair cut) */
        const int64_t x = best_x;
        const int64_t px = pair ? -1 : a[x];
        int64_t bn = 0;
        sub[bn++] = x;
        for (int64_t q = 0; q < bn; q++) {
            int64_t v = sub[q];
            for (int64_t c = cp[F->pos[v]]; c < cp[F->pos[v] + 1]; c++)
                if (a[kids[c]] == v) sub[bn++] = kids[c];
        }
        const int64_t pidb = pf_new_part();
        for (int64_t q = 0; q < bn; q++) __atomic_store_n(&F->part[sub[q]], pidb, __ATOMIC_RELAXED);
        if (!pair) {
            for (int64_t v = px;; v = a[v]) {
                F->SW[v] -= F->SW[x]; F->SD[v] -= F->SD[x];
                F->SO[v] -= F->SO[x]; F->SI[v] -= F->SI[x];
                if (F->root[v]) break;
            }
        }
        for (int64_t q = 0; q < bn; q++) {
            int64_t y = sub[q];
            for (int64_t e = g->uptr[y]; e < g->uptr[y + 1]; e++) {
                int64_t z = g->unbr[e];
                if (pf_part(F, z) != pid) continue;      /* z in the rest */
                double u = g->uu[e];
                F->W[y] -= u;
                F->W[z] -= u;
                /* y's ancestors inside b: stop at x (the new root) */
                for (int64_t v = y;; v = a[v]) { F->SW[v] -= u; if (v == x) break; }
                pf_up(F, z, -u, 0);
                if (!pair) {
                    int64_t l = pf_lca(F, px, z);
                    if (l >= 0) { F->D[l] -= u; pf_up(F, l, -u, 1); }
                }
            }
        }
        a[x] = x;
        F->root[x] = 1;
        if (pair) { a[r0] = r0; F->cycf[r0] = F->cycf[r1] = 0; }
        *changed_out = 1;
        dv_push(gains_out, best_gain);
        sort_u64((uint64_t *)sub, bn);
        int64_t *bpart = (int64_t *)malloc((size_t)bn * sizeof(int64_t));
        memcpy(bpart, sub, (size_t)bn * sizeof(int64_t));
        int64_t *rest = (int64_t *)malloc((size_t)pn * sizeof(int64_t));
        int64_t rn = 0, bi = 0;
        for (int64_t k = 0; k < pn; k++) {
            while (bi < bn && bpart[bi] < mem[k]) bi++;
            if (bi < bn && bpart[bi] == mem[k]) continue;
            rest[rn++] = mem[k];
        }
        free(mem);
        if (sn + 2 > scap) { scap *= 2; stack = (pf_part_t *)realloc(stack, (size_t)scap * sizeof(pf_part_t)); }
        stack[sn++] = (pf_part_t){rest, rn, pid};
        stack[sn++] = (pf_part_t){bpart, bn, pidb};
    }
    free(stack); free(sub); free(cp); free(kids);
    return 0;
}

EXPORT int orc_positive_fast(const orc_graph *g, double m, int64_t *a, const int64_t *comm,
                             int64_t nc, int64_t scc_cap, int64_t *splits, int64_t *unresolved,
                             double *gains_out, int64_t gains_cap, int64_t *n_warn) {
    int64_t n = g->n;
    double *lg = (double *)malloc((size_t)(n ? n : 1) * sizeof(double));
    orc_local_gains(g, m, comm, nc, lg);
    uint8_t *bad = (uint8_t *)calloc((size_t)(nc ? nc : 1), 1);
    int64_t nbad = 0;
    for (int64_t i = 0; i < n; i++) if (lg[i] < 0.0 && !bad[comm[i]]) { bad[comm[i]] = 1; nbad++; }
    free(lg);
    *splits = 0; *unresolved = 0; *n_warn = 0;
    if (nbad == 0) { free(bad); return 0; }
    int64_t *cptr = (int64_t *)calloc((size_t)nc + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) cptr[comm[i] + 1]++;
    for (int64_t c = 0; c < nc; c++) cptr[c + 1] += cptr[c];
    int64_t *cmem = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    {
        int64_t *fill = (int64_t *)malloc((size_t)(nc ? nc : 1) * sizeof(int64_t));
        memcpy(fill, cptr, (size_t)nc * sizeof(int64_t));
        for (int64_t i = 0; i < n; i++) cmem[fill[comm[i]]++] = i;
        free(fill);
    }
    int64_t *blist = (int64_t *)malloc((size_t)nbad * sizeof(int64_t));
    nbad = 0;
    for (int64_t c = 0; c < nc; c++) if (bad[c]) blist[nbad++] = c;
    pf_ctx F;
    memset(&F, 0, sizeof(F));
    F.g = g; F.m = m; F.m2 = m * m; F.a = a;
    F.part = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    F.depth = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    F.pos = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    F.root = (uint8_t *)calloc((size_t)n, 1);
    F.cycf = (uint8_t *)calloc((size_t)n, 1);
    double *buf = (double *)malloc((size_t)n * 6 * sizeof(double));
    F.W = buf; F.D = buf + n; F.SW = buf + 2 * n; F.SD = buf + 3 * n; F.SO = buf + 4 * n; F.SI = buf + 5 * n;
    dvec *gl = (dvec *)calloc((size_t)nbad, sizeof(dvec));
    int64_t *un = (int64_t *)calloc((size_t)nbad, sizeof(int64_t));
    int *ch = (int *)calloc((size_t)nbad, sizeof(int));
    int *lit = (int *)calloc((size_t)nbad, sizeof(int));
    const int64_t BIG = 1 << 16;
    /* small communities in parallel, then the big ones with parallel scans */
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
    for (int64_t k = 0; k < nbad; k++) {
        int64_t c = blist[k];
        int64_t sz = cptr[c + 1] - cptr[c];
        if (sz >= BIG) continue;
        lit[k] = pf_split(&F, cmem + cptr[c], sz, &gl[k], &un[k], &ch[k], 0) < 0;
    }
    for (int64_t k = 0; k < nbad; k++) {
        int64_t c = blist[k];
        int64_t sz = cptr[c + 1] - cptr[c];
        if (sz < BIG) continue;
        lit[k] = pf_split(&F, cmem + cptr[c], sz, &gl[k], &un[k], &ch[k], 1) < 0;
    }
    free(F.part); free(F.depth); free(F.pos); free(F.root); free(F.cycf); free(buf);
    /* communities with a longer cycle: the literal form */
    int any_lit = 0;
    for (int64_t k = 0; k < nbad; k++) any_lit |= lit[k];
    if (any_lit) {
        pos_ctx P;
        memset(&P, 0, sizeof(P));
        P.g = g; P.m = m; P.m2 = m * m; P.a = a; P.scc_cap = scc_cap;
        P.stamp = (int64_t *)calloc((size_t)n, sizeof(int64_t));
        P.in_b = (uint8_t *)calloc((size_t)n, 1);
        P.posof = (int64_t *)malloc((size_t)n * sizeof(int64_t));
        int64_t *seen_pos = (int64_t *)malloc((size_t)n * sizeof(int64_t));
        for (int64_t i = 0; i < n; i++) seen_pos[i] = -1;
        for (int64_t k = 0; k < nbad; k++) {
            if (!lit[k]) continue;
            int64_t c = blist[k];
            P.gains.n = 0; P.unresolved = 0; P.changed = 0;
            split_community(&P, cmem + cptr[c], cptr[c + 1] - cptr[c], seen_pos);
            for (int64_t q = 0; q < P.gains.n; q++) dv_push(&gl[k], P.gains.v[q]);
            un[k] = P.unresolved;
            ch[k] = P.changed;
        }
        *n_warn = P.n_warn;
        free(P.stamp); free(P.in_b); free(P.posof); free(seen_pos);
        dv_free(&P.ws); dv_free(&P.tmp); dv_free(&P.gains);
    }
    int changed = 0;
    int64_t ng = 0;
    for (int64_t k = 0; k < nbad; k++) {
        for (int64_t q = 0; q < gl[k].n; q++) {
            if (gains_out && ng < gains_cap) gains_out[ng] = gl[k].v[q];
            ng++;
        }
        *unresolved += un[k];
        changed |= ch[k];
        dv_free(&gl[k]);
    }
    *splits = ng;
    free(gl); free(un); free(ch); free(lit); free(blist);
    free(cptr); free(cmem); free(bad);
    return changed;
}

/* ------------------------------------------------------------------- PLAN */

/* _best_targets (detector.py:367-418): synchronous best community per node from a
 * frozen snapshot.  S_* are the snapshot aggregates (quality.py:71-79). */
static void plan_rows_raw(const int64_t *uptr, const int64_t *unbr, const double *uu,
                          const double *s_out, const double *s_in, double m, const int64_t *lab,
                          const double *S_out, const double *S_in, int64_t r0, int64_t r1,
                          int64_t row_base, int64_t *cstar) {
    /* rows r0..r1 (global ids); uptr/unbr/uu hold rows row_base.. ; cstar indexed by row */
    const double m2 = m * m;
    int64_t cap = 0;
    int64_t *idx = NULL;
    uint64_t *key = NULL;
    double *wbuf = NULL;
    for (int64_t r = r0; r < r1; r++) {
        int64_t L = lab[r];
        double so = s_out[r], si = s_in[r];
        cstar[r] = L;
        int64_t e0 = uptr[r - row_base], e1 = uptr[r - row_base + 1], d = e1 - e0;
        if (d == 0) continue;
        double t_stay = -(so * (S_in[L] - si) + si * (S_out[L] - so)) / m2;
        if (cap < d) {
            cap = d;
            idx = (int64_t *)realloc(idx, (size_t)cap * sizeof(int64_t));
            key = (uint64_t *)realloc(key, (size_t)cap * sizeof(uint64_t));
            wbuf = (double *)realloc(wbuf, (size_t)cap * sizeof(double));
        }
        /* stable sort entries of the row by community (insertion sort for short rows) */
        for (int64_t k = 0; k < d; k++) { key[k] = (uint64_t)lab[unbr[e0 + k]]; idx[k] = k; }
        if (d <= 32) {
            for (int64_t k = 1; k < d; k++) {
                int64_t v = idx[k]; uint64_t kv = key[v]; int64_t q = k - 1;
                while (q >= 0 && key[idx[q]] > kv) { idx[q + 1] = idx[q]; q--; }
                idx[q + 1] = v;
            }
        } else {
            radix_argsort_u64(key, d, idx);
        }
        double mx = -INFINITY;
        int64_t best_c = -1;
        int64_t k = 0;
        while (k < d) {
            int64_t c = (int64_t)key[idx[k]];
            int64_t q = k, nn = 0;
            while (q < d && (int64_t)key[idx[q]] == c) { wbuf[nn++] = uu[e0 + idx[q]]; q++; }
            double gsum = reduceat_seg(wbuf, nn);
            int own = (c == L);
            double sin_c = S_in[c] - (own ? si : 0.0);
            double sout_c = S_out[c] - (own ? so : 0.0);
            double t = gsum / m - (so * sin_c + si * sout_c) / m2;
            if (own) t_stay = t;
            else if (t > mx) { mx = t; best_c = c; }  /* ascending c: first max kept */
            k = q;
        }
        if (best_c >= 0 && mx > t_stay) cstar[r] = best_c;
    }
    free(idx); free(key); free(wbuf);
}

/* _best_targets (detector.py:367-418): synchronous best community per node from a
 * frozen snapshot.  S_* are the snapshot aggregates (quality.py:71-79). */
static void plan_rows(const orc_graph *g, double m, const int64_t *lab, const double *S_out,
                      const double *S_in, int64_t r0, int64_t r1, int64_t *cstar) {
    plan_rows_raw(g->uptr, g->unbr, g->uu, g->s_out, g->s_in, m, lab, S_out, S_in, r0, r1, 0,
                  cstar);
}

/* Bounded-sample plan over raw arrays (the bench's CPU baseline): rows [r0, r1) whose union
 * rows are given relative to r0. */
EXPORT void orc_plan_sample(const int64_t *uptr, const int64_t *unbr, const double *uu,
                            const double *s_out, const double *s_in, double m, const int64_t *lab,
                            const double *S_out, const double *S_in, int64_t r0, int64_t r1,
                            int64_t *cstar) {
    int64_t n = r1 - r0;
    const int64_t chunk = 2048;
    int64_t nch = (n + chunk - 1) / chunk;
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
    for (int64_t c = 0; c < nch; c++) {
        int64_t a0 = r0 + c * chunk, a1 = a0 + chunk < r1 ? a0 + chunk : r1;
        plan_rows_raw(uptr, unbr, uu, s_out, s_in, m, lab, S_out, S_in, a0, a1, r0, cstar);
    }
}

EXPORT void orc_plan(const orc_graph *g, double m, const int64_t *lab, int64_t nc, int64_t *cstar) {
    double *S_out = (double *)malloc((size_t)(nc ? nc : 1) * sizeof(double));
    double *S_in = (double *)malloc((size_t)(nc ? nc : 1) * sizeof(double));
    int64_t *cnt = (int64_t *)malloc((size_t)(nc ? nc : 1) * sizeof(int64_t));
    aggregates(g, lab, nc, S_out, S_in, cnt);
    int64_t n = g->n;
    const int64_t chunk = 4096;
    int64_t nch = (n + chunk - 1) / chunk;
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
    for (int64_t c = 0; c < nch; c++) {
        int64_t r0 = c * chunk, r1 = r0 + chunk < n ? r0 + chunk : n;
        plan_rows(g, m, lab, S_out, S_in, r0, r1, cstar);
    }
    free(S_out); free(S_in); free(cnt);
}

/* Plan over a row range only, given precomputed aggregates (bounded CPU baseline). */
EXPORT void orc_plan_rows(const orc_graph *g, double m, const int64_t *lab, const double *S_out,
                          const double *S_in, int64_t r0, int64_t r1, int64_t *cstar) {
    int64_t n = r1 - r0;
    const int64_t chunk = 4096;
    int64_t nch = (n + chunk - 1) / chunk;
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
    for (int64_t c = 0; c < nch; c++) {
        int64_t a0 = r0 + c * chunk, a1 = a0 + chunk < r1 ? a0 + chunk : r1;
        plan_rows(g, m, lab, S_out, S_in, a0, a1, cstar);
    }
}

/* ---------------------------------------------------------------------- RNG */

#define RNG_GAMMA 0x9E3779B97F4A7C15ULL
#define RNG_MIX1 0xBF58476D1CE4E5B9ULL
#define RNG_MIX2 0x94D049BB133111EBULL
static uint64_t fin64(uint64_t z) {           /* rng.py:19-23 */
    z = (z ^ (z >> 30)) * RNG_MIX1;
    z = (z ^ (z >> 27)) * RNG_MIX2;
    return z ^ (z >> 31);
}
EXPORT uint64_t orc_mix_key(uint64_t seed, int64_t level, int64_t sweep) {   /* rng.py:26-31 */
    uint64_t s = fin64(seed);
    s = fin64(s + RNG_GAMMA + (uint64_t)level);
    s = fin64(s + RNG_GAMMA + (uint64_t)sweep);
    return s;
}
EXPORT void orc_uniform01(uint64_t seed, int64_t level, int64_t sweep, const int64_t *ids,
                          int64_t k, double *out) {                           /* rng.py:34-43 */
    uint64_t base = orc_mix_key(seed, level, sweep);
    for (int64_t i = 0; i < k; i++) {
        uint64_t z = fin64((uint64_t)ids[i] * RNG_GAMMA + base);
        out[i] = (double)(z >> 11) * 0x1.0p-53;
    }
}

/* ---------------------------------------------------------------- MAXIMAL */

/* maximal_correction (detector.py:457-521).  a: in = forest.a, out = new a.  comm: the
 * forest's canonical labels.  Returns improved; *applied = committed moves. */
EXPORT int orc_maximal(const orc_graph *g, double m, int64_t *a, const int64_t *comm, int64_t nc,
                       uint64_t seed, double accept_prob, int64_t level, int64_t sweep,
                       int64_t *applied_out, double *gains_out, int64_t gains_cap,
                       int64_t *n_cand_out) {
    int64_t n = g->n;
    int64_t *labels = (int64_t *)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
    memcpy(labels, comm, (size_t)n * sizeof(int64_t));
    double *S_out = (double *)malloc((size_t)(nc ? nc : 1) * sizeof(double));
    double *S_in = (double *)malloc((size_t)(nc ? nc : 1) * sizeof(double));
    int64_t *cnt = (int64_t *)malloc((size_t)(nc ? nc : 1) * sizeof(int64_t));
    aggregates(g, labels, nc, S_out, S_in, cnt);
    int64_t *cstar = (int64_t *)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
    orc_plan(g, m, labels, nc, cstar);
    int64_t ncand = 0;
    for (int64_t i = 0; i < n; i++) if (cstar[i] != labels[i]) ncand++;
    if (n_cand_out) *n_cand_out = ncand;
    *applied_out = 0;
    if (ncand == 0) {
        free(labels); free(S_out); free(S_in); free(cnt); free(cstar);
        return 0;
    }
    int64_t *cand = (int64_t *)malloc((size_t)ncand * sizeof(int64_t));
    ncand = 0;
    for (int64_t i = 0; i < n; i++) if (cstar[i] != labels[i]) cand[ncand++] = i;
    double *u01 = (double *)malloc((size_t)ncand * sizeof(double));
    orc_uniform01(seed, level, sweep, cand, ncand, u01);
    /* reverse_assignment (forest.py:70-80): kids ascending per target, self excluded */
    int64_t *rptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) if (a[i] != i) rptr[a[i] + 1]++;
    for (int64_t i = 0; i < n; i++) rptr[i + 1] += rptr[i];
    int64_t *rkids = (int64_t *)malloc((size_t)(rptr[n] ? rptr[n] : 1) * sizeof(int64_t));
    {
        int64_t *fill = (int64_t *)malloc((size_t)n * sizeof(int64_t));
        memcpy(fill, rptr, (size_t)n * sizeof(int64_t));
        for (int64_t i = 0; i < n; i++) if (a[i] != i) rkids[fill[a[i]]++] = i;
        free(fill);
    }
    uint8_t *dirty = (uint8_t *)calloc((size_t)nc, 1);
    uint8_t *in_set = (uint8_t *)calloc((size_t)n, 1);
    uint8_t *seen = (uint8_t *)calloc((size_t)n, 1);
    ivec moved = {0};
    dvec ws = {0}, tmp = {0}, gains = {0};
    int64_t applied = 0;
    int coin_blocked = 0;
    const double m2 = m * m;
    for (int64_t k = 0; k < ncand; k++) {
        int64_t i = cand[k];
        int64_t frm = labels[i], to = cstar[i];
        if (dirty[frm]) continue;
        if (!(u01[k] < accept_prob)) { coin_blocked = 1; continue; }
        if (cnt[to] == 0) continue;
        /* _tail (detector.py:421-437): BFS over the static reverse assignment */
        moved.n = 0;
        iv_push(&moved, i);
        seen[i] = 1;
        for (int64_t qi = 0; qi < moved.n; qi++) {
            int64_t x = moved.v[qi];
            for (int64_t c = rptr[x]; c < rptr[x + 1]; c++) {
                int64_t kk = rkids[c];
                if (!seen[kk]) { seen[kk] = 1; iv_push(&moved, kk); }
            }
        }
        for (int64_t q = 0; q < moved.n; q++) seen[moved.v[q]] = 0;
        /* gain_switch (quality.py:186-219) */
        for (int64_t q = 0; q < moved.n; q++) in_set[moved.v[q]] = 1;
        double w_to = 0.0, w_from = 0.0;
        for (int64_t q = 0; q < moved.n; q++) {
            int64_t x = moved.v[q];
            dv_clear(&ws); dv_clear(&tmp);
            for (int64_t e = g->uptr[x]; e < g->uptr[x + 1]; e++) {
                int64_t z = g->unbr[e];
                int64_t lz = labels[z];
                if (lz == to) dv_push(&ws, g->uu[e]);
                if (lz == frm && !in_set[z]) dv_push(&tmp, g->uu[e]);
            }
            w_to += pw_sum(ws.v, ws.n);
            w_from += pw_sum(tmp.v, tmp.n);
        }
        for (int64_t q = 0; q < moved.n; q++) in_set[moved.v[q]] = 0;
        dv_clear(&tmp);
        for (int64_t q = 0; q < moved.n; q++) dv_push(&tmp, g->s_out[moved.v[q]]);
        double so_b = pw_sum(tmp.v, tmp.n);
        dv_clear(&tmp);
        for (int64_t q = 0; q < moved.n; q++) dv_push(&tmp, g->s_in[moved.v[q]]);
        double si_b = pw_sum(tmp.v, tmp.n);
        double so_t = S_out[to], si_t = S_in[to];
        double d_null = (-S_out[frm] * si_b - so_b * S_in[frm] + so_t * si_b + so_b * si_t
                         + 2.0 * so_b * si_b);
        double gn = (w_to - w_from) / m - d_null / (m * m);
        if (!(gn > 0.0)) continue;
        /* _attach_target (detector.py:440-454) */
        int64_t j = -1;
        double best = 0.0;
        double soi = g->s_out[i], sii = g->s_in[i];
        for (int64_t e = g->uptr[i]; e < g->uptr[i + 1]; e++) {
            int64_t z = g->unbr[e];
            if (labels[z] != to) continue;
            double pg = g->uu[e] / m - (soi * g->s_in[z] + sii * g->s_out[z]) / m2;
            if (j < 0 || pg > best) { best = pg; j = z; }
        }
        if (j < 0) continue;
        a[i] = j;
        for (int64_t q = 0; q < moved.n; q++) labels[moved.v[q]] = to;
        /* move_nodes (quality.py:87-95) */
        S_out[frm] -= so_b; S_in[frm] -= si_b; cnt[frm] -= moved.n;
        S_out[to] += so_b; S_in[to] += si_b; cnt[to] += moved.n;
        dirty[frm] = 1; dirty[to] = 1;
        applied++;
        dv_push(&gains, gn);
    }
    *applied_out = applied;
    if (gains_out) {
        int64_t k = gains.n < gains_cap ? gains.n : gains_cap;
        memcpy(gains_out, gains.v, (size_t)k * sizeof(double));
    }
    free(labels); free(S_out); free(S_in); free(cnt); free(cstar); free(cand); free(u01);
    free(rptr); free(rkids); free(dirty); free(in_set); free(seen);
    iv_free(&moved); dv_free(&ws); dv_free(&tmp); dv_free(&gains);
    return (applied > 0) || coin_blocked;
}

/* ------------------------------------------------------------------- SCORE */

/* score (quality.py:104-118) with resolution: (intra - gamma*null) / m_w. */
EXPORT double orc_score(const orc_graph *g, const int64_t *labels, double gamma) {
    double m = g->m;
    if (m == 0.0) return 0.0;
    dvec v = {0};
    for (int64_t i = 0; i < g->n; i++)
        for (int64_t e = g->out_ptr[i]; e < g->out_ptr[i + 1]; e++)
            if (labels[i] == labels[g->out_dst[e]]) dv_push(&v, g->out_w[e]);
    double intra = pw_sum(v.v, v.n);
    int64_t nc = 0;
    for (int64_t i = 0; i < g->n; i++) if (labels[i] + 1 > nc) nc = labels[i] + 1;
    double *S_out = (double *)calloc((size_t)(nc ? nc : 1), sizeof(double));
    double *S_in = (double *)calloc((size_t)(nc ? nc : 1), sizeof(double));
    for (int64_t i = 0; i < g->n; i++) { S_out[labels[i]] += g->s_out[i]; S_in[labels[i]] += g->s_in[i]; }
    dv_clear(&v);
    for (int64_t c = 0; c < nc; c++) dv_push(&v, S_out[c] * S_in[c] / m);
    double null = pw_sum(v.v, v.n);
    dv_free(&v); free(S_out); free(S_in);
    return (intra - gamma * null) / m;
}

EXPORT double orc_pairwise_sum(const double *a, int64_t n) { return pw_sum(a, n); }
