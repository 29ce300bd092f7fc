/*
 * slm.h -- C ABI of the B200 (sm_100a) Synchronised Louvain Method library (libslm.so).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (synclouvain, pure Python + numpy) has no FFI of its own: its boundary is the Python
 * API `run(graph, RunConfig) -> RunResult` (detector.py:548) over
 * `Graph.from_edges(n, src, dst, w)` (graph.py:84) and the phase functions it calls.
 * Every entry point below replaces one of those reference functions (cited per call);
 * the package paper_1702_04645_b200 binds them with ctypes and re-exposes the reference's
 * Python names, argument meanings and exceptions.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Host arrays are borrowed for the duration of a call.
 *   - Node ids cross the boundary as int64 (graph.py:87-89), weights/gains as fp64.
 *   - Every call returns SLM_OK (0) or a negative code; slm_last_error(ctx) describes it.
 *     SLM_EINVAL maps to the reference's ValueError, the others to RuntimeError.
 *   - Calls are synchronous (the context's stream is synchronised before return) and a
 *     context is single-threaded.  Device state stays resident between calls: the current
 *     hierarchy level's graph and assignment forest live on the GPU, and only labels and
 *     scalars cross the boundary when the caller asks for them.
 *   - Output pointers documented as nullable may be NULL to skip the device->host copy.
 */
#ifndef SLM_H
#define SLM_H

#include <stdint.h>

#if defined(__GNUC__)
#define SLM_API __attribute__((visibility("default")))
#else
#define SLM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SLM_OK 0
#define SLM_EINVAL (-1)
#define SLM_ECUDA (-2)
#define SLM_ENOMEM (-3)
#define SLM_ESTATE (-4)
#define SLM_EUNSUP (-5)

typedef struct slm_ctx slm_ctx;

/* RunConfig (detector.py:22-40) minus threads (meaningless on the GPU), plus resolution. */
typedef struct {
    uint64_t seed;            /* RunConfig.seed, default 0 */
    double accept_prob;       /* RunConfig.accept_prob, default 0.5, in (0, 1] */
    int64_t max_outer_iters;  /* RunConfig.max_outer_iters, default 100 */
    int64_t scc_cut_cap;      /* RunConfig.scc_cut_cap, default 10000 */
    double resolution;        /* gamma; gains use m_w / gamma */
} slm_config;

/* ---- context ------------------------------------------------------------------- */
SLM_API slm_ctx *slm_create(int device);
SLM_API void slm_destroy(slm_ctx *ctx);
SLM_API const char *slm_last_error(slm_ctx *ctx);
SLM_API void *slm_stream(slm_ctx *ctx);                 /* cudaStream_t of the context */
SLM_API int slm_sync(slm_ctx *ctx);

/* ---- graph ----------------------------------------------------------------------- */
/* Graph.from_edges (graph.py:84-116) + neighbor_union (graph.py:127-175) + strengths
 * (graph.py:257-263): canonical CSR, union, strengths and m_w on the device.  Becomes
 * hierarchy level 0 and resets the level counter. */
SLM_API int slm_build_graph(slm_ctx *ctx, int64_t n, const int64_t *src, const int64_t *dst,
                    const double *w, int64_t nedges);
/* Same from device-resident int32 ids / fp64 weights (no host copy). */
SLM_API int slm_build_graph_device(slm_ctx *ctx, int64_t n, const int32_t *d_src, const int32_t *d_dst,
                           const double *d_w, int64_t nedges);
/* Sizes of the current level: nodes, merged CSR entries, union entries, m_w, flags
 * (bit0: symmetric W, bit1: integer weights, bit2: the plan sweep runs the exact uint32
 * group-sum path; otherwise fp64 sums, exact for integers, or the sorted reference-order
 * form for real-valued weights). */
SLM_API int slm_graph_info(slm_ctx *ctx, int64_t *n, int64_t *ne, int64_t *ue, double *m_w,
                   int32_t *flags);
SLM_API int slm_get_csr(slm_ctx *ctx, int64_t *out_ptr, int64_t *out_dst, double *out_w);
/* NeighborUnion ptr/nbr and w_out + w_in (graph.py:46-60) */
SLM_API int slm_get_union(slm_ctx *ctx, int64_t *ptr, int64_t *nbr, double *u);
SLM_API int slm_get_strengths(slm_ctx *ctx, double *s_out, double *s_in);
/* Union rows [r0, r1): ptr_out has r1-r0+1 offsets relative to row r0; nbr_out / u_out
 * nullable (call once with NULL to size them from ptr_out[r1-r0]). */
SLM_API int slm_get_union_rows(slm_ctx *ctx, int64_t r0, int64_t r1, int64_t *ptr_out,
                               int64_t *nbr_out, double *u_out);
/* Canonical CSR rows [r0, r1) (Graph.out_ptr / out_dst / out_w slices, graph.py:97-110), in
 * the same convention as slm_get_union_rows (bounded downloads of 1e9-entry graphs). */
SLM_API int slm_get_csr_rows(slm_ctx *ctx, int64_t r0, int64_t r1, int64_t *ptr_out,
                             int64_t *dst_out, double *w_out);
SLM_API int slm_set_resolution(slm_ctx *ctx, double gamma);

/* ---- phases (current level) ----------------------------------------------------- */
/* find_assignment (detector.py:149-158); a_out nullable. */
SLM_API int slm_assign(slm_ctx *ctx, int64_t *a_out);
/* Load an assignment map (differential tests / resume); builds the forest. */
SLM_API int slm_set_assignment(slm_ctx *ctx, const int64_t *a);
/* extract_components (forest.py:43-67) of the device assignment; outputs nullable. */
SLM_API int slm_components(slm_ctx *ctx, int64_t *comm_out, uint8_t *on_cycle_out, int64_t *n_comms);
/* Current forest (a, comm, on_cycle); outputs nullable. */
SLM_API int slm_get_forest(slm_ctx *ctx, int64_t *a_out, int64_t *comm_out, uint8_t *on_cycle_out,
                   int64_t *n_comms);
/* CommunityAggregates.from_labels (quality.py:71-79) of the current forest. */
SLM_API int slm_get_aggregates(slm_ctx *ctx, double *S_out, double *S_in, int64_t *count);
/* local_gains (quality.py:170-183) of the current forest. */
SLM_API int slm_local_gains(slm_ctx *ctx, double *lg_out);
/* positive_correction (detector.py:338-362); gains_out (nullable) receives up to
 * gains_cap gains in the reference's order. */
SLM_API int slm_positive(slm_ctx *ctx, const slm_config *cfg, int64_t *splits, int64_t *unresolved,
                 int32_t *changed, double *gains_out, int64_t gains_cap);
/* _best_targets over all rows (detector.py:367-418): the local-move sweep.  comm_in
 * (nullable) replaces the forest labels as the snapshot (must be dense, with the
 * aggregates recomputed from it); cstar_out nullable. */
SLM_API int slm_plan_sweep(slm_ctx *ctx, const int64_t *comm_in, int64_t *cstar_out);
/* Bench helpers: enqueue one plan sweep on the context stream without synchronising or
 * copying (bin_mask bit b = degree bin b of 6 (<=32, <=256, <=1024, <=4096, <=16383,
 * larger), bit 6 = label copy for rows without entries; 127 = the full sweep); count the
 * distinct (node, community) groups G of the snapshot and the rows / union entries of each
 * of the 6 degree bins; read the last plan's targets. */
SLM_API int slm_plan_sweep_async(slm_ctx *ctx, int32_t bin_mask);
SLM_API int slm_plan_groups(slm_ctx *ctx, int64_t *groups, int64_t *bin_rows, int64_t *bin_entries);
SLM_API int slm_get_cstar(slm_ctx *ctx, int64_t *cstar_out);
/* Diagnostics: device ms of a pure stream of the union (mode 0), + neighbour-label gathers
 * (1), + community-strength gathers (2) -- the memory-system floor of the sweep; modes 3-5:
 * the same over the degree-ordered sweep view. */
SLM_API int slm_debug_sweep_floor(slm_ctx *ctx, int32_t mode, double *ms);
/* run() of detector.py:548-653 in one call (no host round trip per phase): the whole
 * level loop on the current graph with the reference's stop rules and the exact
 * fast-forward.  stats[5] = accepted_moves, accepted_splits, unresolved_negative, skipped
 * POSITIVE calls, levels stopped at max_outer_iters; phase_s[5] = wall seconds of assign,
 * components, positive, maximal, aggregate (nullable).  Per-level results via
 * slm_run_level (labels_out nullable; plan_path 0 = uint32 fast path, 1 = fp64 on integer
 * sums, 2 = sorted reference order, plus 8 when the level stopped at max_outer_iters). */
SLM_API int slm_run(slm_ctx *ctx, const slm_config *cfg, int64_t *n_levels, int64_t *stats,
                    double *phase_s);
SLM_API int slm_run_level(slm_ctx *ctx, int64_t t, int64_t *n_nodes, int64_t *sweeps,
                          int32_t *plan_path, int64_t *labels_out);

/* ---- the rest of the reference's hot-path API (slm_surface.cu) ------------------- */
/* CommunityAggregates.from_labels (quality.py:71-79) over caller strengths: S_out / S_in
 * by sequential per-community sums in node order (np.bincount), member counts. */
SLM_API int slm_community_sums(slm_ctx *ctx, int64_t n, const int64_t *labels, int64_t n_comms,
                               const double *s_out, const double *s_in, double *S_out,
                               double *S_in, int64_t *count);
/* gain_switch (quality.py:186-219) on the current level graph: exact score change of
 * relabeling nodes[0..k) from frm to to (to < 0: a fresh empty community); agg4 =
 * {S_out[frm], S_in[frm], S_out[to], S_in[to]} of the caller's aggregates; m = st.m_w. */
SLM_API int slm_gain_switch(slm_ctx *ctx, const int64_t *labels, const int64_t *nodes, int64_t k,
                            int64_t frm, int64_t to, const double *agg4, double m, double *gain);
/* reverse_assignment (forest.py:70-80): ptr_out[n+1], kids_out[n] (children j != i with
 * a[j] == i, ascending), *n_kids = ptr_out[n]. */
SLM_API int slm_reverse_assignment(slm_ctx *ctx, int64_t n, const int64_t *a, int64_t *ptr_out,
                                   int64_t *kids_out, int64_t *n_kids);
/* NeighborUnion.w_out / w_in (graph.py:46-60, 151-175) of the current level: W(i, j) and
 * W(j, i) per union entry (w_out + w_in == the stored u bit for bit). */
SLM_API int slm_get_union_split(slm_ctx *ctx, double *w_out, double *w_in);
/* canonicalize_labels (graph.py:283-291): dense labels ordered by first occurrence. */
SLM_API int slm_canonicalize_labels(slm_ctx *ctx, int64_t n, const int64_t *labels, int64_t *out,
                                    int64_t *n_comms);
/* aggregate(graph, labels) (graph.py:266-280) of src's current level graph, built on the
 * device as level 0 of ctx (same device; labels dense 0..n_comms-1). */
SLM_API int slm_build_aggregate(slm_ctx *ctx, slm_ctx *src, const int64_t *labels,
                                int64_t n_comms);

/* Diagnostics of the device primitives (slm_prim.cu), on host arrays, in place:
 * slm_debug_sort: stable LSD radix sort by bits [0, end_bit) of (kind 0) uint64 keys with
 * double values or (kind 1) uint32 keys with int32 values; *ms = device time of the sort.
 * slm_debug_scan: exclusive prefix sum, kind 0 int64, 1 int32, 2 int32 -> int64, 3 double,
 * 4 int32 restarting at every change of keys[] (keys nullable otherwise). */
SLM_API int slm_debug_sort(slm_ctx *ctx, int32_t kind, void *keys, void *vals, int64_t n,
                           int32_t end_bit, double *ms);
SLM_API int slm_debug_scan(slm_ctx *ctx, int32_t kind, const void *in, void *out,
                           const uint32_t *keys, int64_t n);
/* maximal_correction (detector.py:457-521) for (level, sweep); gains_out nullable. */
SLM_API int slm_maximal(slm_ctx *ctx, const slm_config *cfg, int64_t level, int64_t sweep,
                int32_t *improved, int64_t *applied, double *gains_out, int64_t gains_cap);
/* aggregate (graph.py:266-280) by the current forest's labels: the coarse graph becomes
 * the current level. */
SLM_API int slm_aggregate(slm_ctx *ctx);
/* score (quality.py:104-118) with resolution: (intra - gamma*null)/m_w.  on_original != 0
 * scores the level-0 graph, else the current level. */
SLM_API int slm_score(slm_ctx *ctx, int32_t on_original, const int64_t *labels, double gamma,
              double *q_out);
/* uniform01 (rng.py:34-43) with parts = (level, sweep), computed on the device. */
SLM_API int slm_uniform01(slm_ctx *ctx, uint64_t seed, int64_t level, int64_t sweep, const int64_t *ids,
                  int64_t k, double *out);
/* Phase timers (enabled by SLM_PROFILE=1, which synchronises at phase boundaries): ms per
 * phase in the order plan, candidates, spec, walk, components, aggregates, layout,
 * positive-local-gains, positive-small, positive-giant, assign, aggregate; then (always
 * measured) host ms in cudaMalloc / cudaFree, their count, and host ms spent building the
 * levels' sweep views. */
SLM_API int slm_phase_times(slm_ctx *ctx, double *ms, int32_t nmax, int32_t reset);
/* Diagnostics of the last slm_maximal: candidates, commit rounds. */
SLM_API int slm_last_commit_stats(slm_ctx *ctx, int64_t *candidates, int64_t *rounds);

/* ---- synthetic inputs (BASELINE.json configs) ------------ */
/* Device generators: symmetrised R-MAT with permuted ids, self-loops dropped (weight_mode
 * 0 = unit, 1 = uniform integers in [1, 100]), and the random geometric graph in the unit
 * square, generated in HBM straight into the level-0 build.  Their host twins (the same edge
 * multisets, for the oracle and the tests) live outside this library, in workloads/gen_host.c. */
SLM_API int slm_build_rmat(slm_ctx *ctx, int scale, int edge_factor, double a, double b, double c,
                   uint64_t seed, int weight_mode);
SLM_API int slm_build_rgg(slm_ctx *ctx, int64_t n, double radius, uint64_t seed);
/* Pair-model graphs generated in HBM, one Bernoulli draw per node pair i < j (both
 * directions, unit weights): mode 0 = planted-partition SBM (blocks of n / blocks
 * consecutive ids, p_in / p_out); mode 1 = Chung-Lu DC-SBM over per-node parameters
 * (community comm[i], kin[i], kout[i], per-community K, total O; p = min(1, kin_i kin_j / K_c)
 * inside a community, min(1, kout_i kout_j / O) across).  Host twin: workloads/gen_host.c. */
SLM_API int slm_build_pairs(slm_ctx *ctx, int32_t mode, int64_t n, int64_t blocks, double p_in,
                            double p_out, const int32_t *comm, const double *kin,
                            const double *kout, const double *K, int64_t n_comms, double O,
                            uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif /* SLM_H */
