"""Generate the golden parity fixtures from the reference itself (run in the build container).

Imports the unmodified reference from /root/reference/pkg/src (and its test-suite graph
helper from /root/reference/pkg/tests/oracles.py) and records, for small seeded inputs,
the outputs of every hot-path phase and of full runs.  The fixtures are committed; the
reference tree does not exist on the GPU box and is never read at test time.

    python tests/golden/make_golden.py
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import synclouvain as S  # noqa: E402
from synclouvain import rng as R  # noqa: E402
from oracles import random_edges  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def edges_arrays(edges):
    return (np.array([e[0] for e in edges], np.int64), np.array([e[1] for e in edges], np.int64),
            np.array([e[2] for e in edges], np.float64))


def record_case(out, key, n, src, dst, w, seed, p):
    G = S.Graph.from_edges(n, src, dst, w)
    st = S.strengths(G)
    U = G.neighbor_union()
    out[f"{key}/n"] = np.int64(n)
    out[f"{key}/src"], out[f"{key}/dst"], out[f"{key}/w"] = src, dst, w
    out[f"{key}/seed"], out[f"{key}/p"] = np.int64(seed), np.float64(p)
    out[f"{key}/out_ptr"], out[f"{key}/out_dst"], out[f"{key}/out_w"] = G.out_ptr, G.out_dst, G.out_w
    out[f"{key}/uptr"], out[f"{key}/unbr"], out[f"{key}/uu"] = U.ptr, U.nbr, U.w_out + U.w_in
    out[f"{key}/s_out"], out[f"{key}/s_in"], out[f"{key}/m_w"] = st.s_out, st.s_in, np.float64(st.m_w)
    a = S.find_assignment(G, st)
    out[f"{key}/assign"] = a
    f = S.extract_components(a)
    out[f"{key}/comm0"], out[f"{key}/on_cycle0"] = f.comm, f.on_cycle
    cfg = S.RunConfig(seed=seed, accept_prob=p)
    agg = S.CommunityAggregates.from_labels(st, f.comm, f.n_comms)
    out[f"{key}/lg0"] = S.local_gains(G, st, f.comm, agg)
    f2, sp, un, gains = S.positive_correction(G, st, f, cfg, None)
    out[f"{key}/pos_a"], out[f"{key}/pos_comm"] = f2.a, f2.comm
    out[f"{key}/pos_stats"] = np.array([sp, un], np.int64)
    out[f"{key}/pos_gains"] = np.array(gains, np.float64)
    from synclouvain.detector import _best_targets
    agg2 = S.CommunityAggregates.from_labels(st, f2.comm, f2.n_comms)
    out[f"{key}/cstar"] = _best_targets(G, st, f2.comm, agg2, 0, n)
    f3, imp, app, g3 = S.maximal_correction(G, st, f2, cfg, 0, 0, None)
    out[f"{key}/max_a"], out[f"{key}/max_comm"] = f3.a, f3.comm
    out[f"{key}/max_stats"] = np.array([int(imp), app], np.int64)
    out[f"{key}/max_gains"] = np.array(g3, np.float64)
    res = S.run(G, cfg)
    out[f"{key}/nlevels"] = np.int64(len(res.hierarchy.levels))
    for t, lv in enumerate(res.hierarchy.levels):
        out[f"{key}/level{t}"] = lv
    out[f"{key}/flat"] = res.hierarchy.flat
    out[f"{key}/final_score"] = np.float64(res.final_score)
    out[f"{key}/sweeps"] = np.array(res.stats.sweeps_per_level, np.int64)
    out[f"{key}/run_stats"] = np.array([res.stats.accepted_moves, res.stats.accepted_splits,
                                        res.stats.unresolved_negative], np.int64)


def main():
    out = {}
    cases = []
    rng = np.random.default_rng(20240811)   # the reference suite's fixture seed
    for t in range(16):
        n = int(rng.integers(4, 70))
        dens = float(rng.uniform(0.06, 0.35))
        edges = random_edges(rng, n, density=dens, dyadic=(t % 2 == 0), self_loops=(t % 3 == 0))
        cases.append((f"rand{t:02d}", n, edges, t, [0.5, 1.0, 0.3][t % 3]))
    # integer weights: undirected multigraph with summed duplicates (C3/C5 shape in miniature)
    for t in range(6):
        n = int(rng.integers(20, 120))
        m = int(n * rng.uniform(2, 6))
        s = rng.integers(0, n, m)
        d = rng.integers(0, n, m)
        keep = s != d
        w = rng.integers(1, 101, m).astype(float)
        edges = [(int(a), int(b), float(x)) for a, b, x in zip(s[keep], d[keep], w[keep])]
        edges = edges + [(b, a, x) for a, b, x in edges]
        cases.append((f"int{t:02d}", n, edges, 100 + t, 0.5))
    for key, n, edges, seed, p in cases:
        src, dst, w = edges_arrays(edges)
        record_case(out, key, n, src, dst, w, seed, p)
    out["cases"] = np.array([c[0] for c in cases])
    # RNG known answers (rng.py:26-43)
    ids = np.array([0, 1, 2, 1000000, 16777215, 123456789012], np.int64)
    out["rng/ids"] = ids
    out["rng/u_0_0_0"] = R.uniform01(0, (0, 0), ids)
    out["rng/u_11_2_5"] = R.uniform01(11, (2, 5), ids)
    out["rng/mix_0_0_0"] = np.uint64(R.mix_key(0, 0, 0))
    np.savez_compressed(os.path.join(HERE, "reference_phases.npz"), **out)
    print("wrote", len(cases), "cases")


if __name__ == "__main__" and "--configs" not in sys.argv and "--surface" not in sys.argv:
    main()


def configs():
    """Full-run fixtures of config 1 and scaled stand-ins of configs 3-5 (same generators)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    import workloads as GN
    out = {}
    specs = [("c1_sbm", GN.generate("c1_sbm")),
             ("c2_dcsbm_small", GN.dcsbm(n=3000, k=20, size_lo=50, size_hi=300, seed=1)),
             ("c3_rmat10", GN.rmat(10, 16, 0, 2)),
             ("c4_rgg4096", GN.rgg(4096, 8.0, 3)),
             ("c5_rmat10w", GN.rmat(10, 8, 1, 4))]
    for key, (n, s, d, w) in specs:
        G = S.Graph.from_edges(n, s, d, w)
        res = S.run(G, S.RunConfig(seed=0))
        out[f"{key}/n"] = np.int64(n)
        out[f"{key}/edges_sha"] = np.array([hash_edges(s, d, w)])
        out[f"{key}/nlevels"] = np.int64(len(res.hierarchy.levels))
        for t, lv in enumerate(res.hierarchy.levels):
            out[f"{key}/level{t}"] = lv
        out[f"{key}/final_score"] = np.float64(res.final_score)
        out[f"{key}/sweeps"] = np.array(res.stats.sweeps_per_level, np.int64)
        out[f"{key}/run_stats"] = np.array([res.stats.accepted_moves, res.stats.accepted_splits,
                                            res.stats.unresolved_negative], np.int64)
        print(key, n, len(s), res.stats.sweeps_per_level, res.final_score)
    np.savez_compressed(os.path.join(HERE, "reference_configs.npz"), **out)


def hash_edges(s, d, w):
    import hashlib
    h = hashlib.sha256()
    for a in (np.asarray(s, np.int64), np.asarray(d, np.int64), np.asarray(w, np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


if __name__ == "__main__" and "--configs" in sys.argv:
    configs()


def surface():
    """reference_surface.npz: the rest of the hot-path API surface on the same golden graphs --
    NeighborUnion.w_out / w_in, reverse_assignment, canonicalize_labels,
    CommunityAggregates.from_labels, gain_switch (incl. to=None) and aggregate()."""
    from synclouvain.forest import reverse_assignment
    from synclouvain.graph import aggregate, canonicalize_labels
    from synclouvain.quality import gain_switch
    ph = np.load(os.path.join(HERE, "reference_phases.npz"))
    out = {}
    rng = np.random.default_rng(5150)
    for key in [str(c) for c in ph["cases"]]:
        n = int(ph[f"{key}/n"])
        G = S.Graph.from_edges(n, ph[f"{key}/src"], ph[f"{key}/dst"], ph[f"{key}/w"])
        st = S.strengths(G)
        U = G.neighbor_union()
        out[f"{key}/w_out"], out[f"{key}/w_in"] = U.w_out, U.w_in
        for tag in ("assign", "pos_a", "max_a"):
            p, kids = reverse_assignment(ph[f"{key}/{tag}"])
            out[f"{key}/rev_{tag}_ptr"], out[f"{key}/rev_{tag}_kids"] = p, kids
        raw = rng.integers(-7, 3 * n, n)
        out[f"{key}/canon_in"] = raw
        out[f"{key}/canon_out"] = canonicalize_labels(raw)
        comm = ph[f"{key}/pos_comm"]
        nc = int(comm.max()) + 1
        agg = S.CommunityAggregates.from_labels(st, comm, nc)
        out[f"{key}/agg_s_out"], out[f"{key}/agg_s_in"], out[f"{key}/agg_count"] = \
            agg.s_out, agg.s_in, agg.count
        gs = []
        for t in range(8):
            frm = int(comm[rng.integers(0, n)])
            mem = np.flatnonzero(comm == frm)
            k = int(rng.integers(1, mem.size + 1))
            nodes = np.sort(rng.choice(mem, size=k, replace=False))
            to = None if t % 4 == 3 else int(rng.integers(0, nc))
            g = gain_switch(G, st, comm, agg, nodes, frm, to)
            gs.append((frm, -1 if to is None else to, k, g))
            out[f"{key}/gs{t}_nodes"] = nodes
        out[f"{key}/gs"] = np.array(gs, np.float64)
        H = aggregate(G, comm)
        out[f"{key}/agg_graph_ptr"], out[f"{key}/agg_graph_dst"], out[f"{key}/agg_graph_w"] = \
            H.out_ptr, H.out_dst, H.out_w
    out["cases"] = ph["cases"]
    np.savez_compressed(os.path.join(HERE, "reference_surface.npz"), **out)
    print("wrote surface fixtures")


if __name__ == "__main__" and "--surface" in sys.argv:
    surface()
