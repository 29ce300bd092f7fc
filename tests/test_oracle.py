"""The C oracle (oracle/slm_oracle.c) pinned against the reference.

CPU-only.  Every phase of every golden case (tests/golden/reference_phases.npz, produced by
the unmodified reference via tests/golden/make_golden.py) must be reproduced bit for bit,
including real-valued weights (the oracle keeps numpy's summation orders).  Where the
reference tree exists (the build container) the oracle is also run against the live
reference on fresh seeded graphs.
"""

import os
import sys

import numpy as np
import pytest

from tests.conftest import REFERENCE_SRC, case_edges, case_names


def _cases(golden):
    return case_names(golden)


def test_rng_known_answers(oracle, golden):
    ids = golden["rng/ids"]
    assert oracle.mix_key(0, 0, 0) == int(golden["rng/mix_0_0_0"])
    np.testing.assert_array_equal(oracle.uniform01(0, 0, 0, ids), golden["rng/u_0_0_0"])
    np.testing.assert_array_equal(oracle.uniform01(11, 2, 5, ids), golden["rng/u_11_2_5"])
    # SURVEY.md §8(c) values generated from rng.py
    assert oracle.mix_key(0, 0, 0) == 0xa706dd2f4d197e6f
    np.testing.assert_array_equal(
        oracle.uniform01(0, 0, 0, [0, 1, 2, 1000000, 16777215]),
        [0.7054856102290845, 0.13870941014555427, 0.9711020828012883, 0.1639810039912002,
         0.5766305475546153])


def test_pairwise_sum_matches_numpy(oracle):
    rng = np.random.default_rng(5)
    for n in [0, 1, 7, 8, 9, 127, 128, 129, 1000, 4097, 100003]:
        x = rng.uniform(0.1, 3.0, n)
        assert oracle.pairwise_sum(x) == float(x.sum())


def test_graph_build_matches_reference(oracle, golden):
    for key in _cases(golden):
        n, s, d, w = case_edges(golden, key)
        g = oracle.OGraph.from_edges(n, s, d, w)
        p, dst, ww = g.csr()
        np.testing.assert_array_equal(p, golden[f"{key}/out_ptr"])
        np.testing.assert_array_equal(dst, golden[f"{key}/out_dst"])
        np.testing.assert_array_equal(ww, golden[f"{key}/out_w"])
        up, un, uu = g.union()
        np.testing.assert_array_equal(up, golden[f"{key}/uptr"])
        np.testing.assert_array_equal(un, golden[f"{key}/unbr"])
        np.testing.assert_array_equal(uu, golden[f"{key}/uu"])
        so, si, m = g.strengths()
        np.testing.assert_array_equal(so, golden[f"{key}/s_out"])
        np.testing.assert_array_equal(si, golden[f"{key}/s_in"])
        assert m == float(golden[f"{key}/m_w"])


def test_phases_match_reference(oracle, golden):
    for key in _cases(golden):
        n, s, d, w = case_edges(golden, key)
        seed, p = int(golden[f"{key}/seed"]), float(golden[f"{key}/p"])
        g = oracle.OGraph.from_edges(n, s, d, w)
        a = oracle.find_assignment(g)
        np.testing.assert_array_equal(a, golden[f"{key}/assign"], err_msg=key)
        comm, nc, oc = oracle.extract_components(a)
        np.testing.assert_array_equal(comm, golden[f"{key}/comm0"])
        np.testing.assert_array_equal(oc, golden[f"{key}/on_cycle0"])
        np.testing.assert_array_equal(oracle.local_gains(g, comm, nc), golden[f"{key}/lg0"])
        a2, ch, sp, un, gains, _ = oracle.positive_correction(g, a, comm, nc)
        np.testing.assert_array_equal(a2, golden[f"{key}/pos_a"], err_msg=key)
        assert [sp, un] == list(golden[f"{key}/pos_stats"])
        np.testing.assert_array_equal(gains, golden[f"{key}/pos_gains"])
        comm2, nc2, _ = oracle.extract_components(a2)
        np.testing.assert_array_equal(comm2, golden[f"{key}/pos_comm"])
        np.testing.assert_array_equal(oracle.best_targets(g, comm2, nc2), golden[f"{key}/cstar"])
        a3, imp, app, g3, _ = oracle.maximal_correction(g, a2, comm2, nc2, seed, p, 0, 0)
        np.testing.assert_array_equal(a3, golden[f"{key}/max_a"], err_msg=key)
        assert [int(imp), app] == list(golden[f"{key}/max_stats"])
        np.testing.assert_array_equal(g3, golden[f"{key}/max_gains"])


def test_full_runs_match_reference(oracle, golden):
    for key in _cases(golden):
        n, s, d, w = case_edges(golden, key)
        seed, p = int(golden[f"{key}/seed"]), float(golden[f"{key}/p"])
        r = oracle.run(n, s, d, w, seed=seed, accept_prob=p)
        assert len(r.levels) == int(golden[f"{key}/nlevels"]), key
        for t, lv in enumerate(r.levels):
            np.testing.assert_array_equal(lv, golden[f"{key}/level{t}"])
        np.testing.assert_array_equal(r.flat, golden[f"{key}/flat"])
        assert r.final_score == float(golden[f"{key}/final_score"])
        assert r.sweeps_per_level == list(golden[f"{key}/sweeps"])
        assert [r.accepted_moves, r.accepted_splits, r.unresolved_negative] == \
            list(golden[f"{key}/run_stats"])


def test_config_fixtures(oracle, golden_configs):
    import workloads as GN
    from tests.golden.make_golden import hash_edges
    specs = {"c1_sbm": lambda: GN.generate("c1_sbm"),
             "c2_dcsbm_small": lambda: GN.dcsbm(n=3000, k=20, size_lo=50, size_hi=300, seed=1),
             "c3_rmat10": lambda: GN.rmat(10, 16, 0, 2),
             "c4_rgg4096": lambda: GN.rgg(4096, 8.0, 3),
             "c5_rmat10w": lambda: GN.rmat(10, 8, 1, 4)}
    G = golden_configs
    for key, fn in specs.items():
        n, s, d, w = fn()
        assert hash_edges(s, d, w) == str(G[f"{key}/edges_sha"][0]), key
        r = oracle.run(n, s, d, w, seed=0)
        assert len(r.levels) == int(G[f"{key}/nlevels"])
        for t, lv in enumerate(r.levels):
            np.testing.assert_array_equal(lv, G[f"{key}/level{t}"])
        assert r.final_score == float(G[f"{key}/final_score"])
        assert r.sweeps_per_level == list(G[f"{key}/sweeps"])
        assert [r.accepted_moves, r.accepted_splits, r.unresolved_negative] == \
            list(G[f"{key}/run_stats"])


# ------------------------------------------------------------- live reference

@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference tree not present (GPU box)")
    sys.path.insert(0, REFERENCE_SRC)
    import synclouvain
    return synclouvain


def test_oracle_vs_live_reference_random(oracle, ref):
    sys.path.insert(0, "/root/reference/pkg/tests")
    from oracles import random_edges
    rng = np.random.default_rng(424242)
    for t in range(25):
        n = int(rng.integers(2, 90))
        edges = random_edges(rng, n, density=float(rng.uniform(0.03, 0.4)), dyadic=bool(t % 2),
                             self_loops=bool(t % 4 == 0))
        s = np.array([e[0] for e in edges], np.int64)
        d = np.array([e[1] for e in edges], np.int64)
        w = np.array([e[2] for e in edges], np.float64)
        cfg = ref.RunConfig(seed=t, accept_prob=[0.5, 1.0, 0.25][t % 3])
        rr = ref.run(ref.Graph.from_edges(n, s, d, w), cfg)
        ro = oracle.run(n, s, d, w, seed=t, accept_prob=cfg.accept_prob)
        assert len(rr.hierarchy.levels) == len(ro.levels)
        for x, y in zip(rr.hierarchy.levels, ro.levels):
            np.testing.assert_array_equal(x, y)
        assert rr.final_score == ro.final_score
        assert rr.stats.sweeps_per_level == ro.sweeps_per_level


def test_oracle_resolution_matches_patched_reference(oracle, ref, monkeypatch):
    """gamma in {0.5, 2}: the reference with m_w -> m_w/gamma."""
    import workloads as GN
    import synclouvain.detector as D
    n, s, d, w = GN.generate("c1_sbm")
    for gamma in (0.5, 2.0):
        orig = D.strengths

        def patched(g, _o=orig, _gm=gamma):
            st = _o(g)
            return ref.Strengths(st.s_out, st.s_in, st.m_w / _gm)
        monkeypatch.setattr(D, "strengths", patched)
        rr = ref.run(ref.Graph.from_edges(n, s, d, w), ref.RunConfig(seed=0))
        monkeypatch.setattr(D, "strengths", orig)
        ro = oracle.run(n, s, d, w, seed=0, resolution=gamma)
        assert len(rr.hierarchy.levels) == len(ro.levels)
        for x, y in zip(rr.hierarchy.levels, ro.levels):
            np.testing.assert_array_equal(x, y)
        assert rr.stats.sweeps_per_level == ro.sweeps_per_level


def test_oracle_kats():
    """Reference known answers (test_detector.py / test_quality.py) through the oracle."""
    from oracle import oracle as O
    tri = [(0, 1, 1.0), (1, 2, 1.0), (2, 0, 1.0), (3, 4, 1.0), (4, 5, 1.0), (5, 3, 1.0)]
    s, d, w = (np.array(x) for x in zip(*tri))
    g = O.OGraph.from_edges(6, s, d, w)
    np.testing.assert_array_equal(O.find_assignment(g), [1, 0, 0, 4, 3, 3])
    assert O.score(g, [0, 0, 0, 1, 1, 1]) == 0.5
    assert abs(O.score(g, np.arange(6)) - (-1.0 / 6.0)) < 1e-15
    r = O.run(6, s, d, w, accept_prob=1.0)
    assert [lv.tolist() for lv in r.levels] == [[0, 0, 0, 1, 1, 1], [0, 1]]
    assert r.final_score == 0.5
    g2 = O.OGraph.from_edges(2, [0], [1], [1.0])
    np.testing.assert_array_equal(O.find_assignment(g2), [0, 1])
    k4 = [(i, j, 1.0) for i in range(4) for j in range(4) if i != j]
    s, d, w = (np.array(x) for x in zip(*k4))
    np.testing.assert_array_equal(O.run(4, s, d, w, accept_prob=1.0).flat, [0, 0, 0, 0])
    # pendant detach (test_detector.py:50-78)
    e = [(0, 1, 1.0), (1, 2, 1.0), (2, 0, 1.0), (3, 0, 0.5), (3, 4, 5.0)]
    s, d, w = (np.array(x) for x in zip(*e))
    g = O.OGraph.from_edges(5, s, d, w)
    a = np.array([1, 2, 0, 0, 4])
    comm, nc, _ = O.extract_components(a)
    a2, ch, sp, un, gains, _ = O.positive_correction(g, a, comm, nc)
    assert sp == 1 and un == 0 and gains[0] > 0 and a2[3] == 3
    np.testing.assert_array_equal(O.extract_components(a2)[0], [0, 0, 0, 1, 2])
    with pytest.raises(ValueError):
        O.OGraph.from_edges(2, [0], [2], [1.0])
    with pytest.raises(ValueError):
        O.OGraph.from_edges(2, [0], [1], [0.0])


# ------------------------------------------------ fast POSITIVE vs the literal form

def _loop_compare_positive(O, n, s, d, w, seed=0, accept_prob=0.5, resolution=1.0, sweeps=6):
    """Run the level loop (detector.py:573-641, capped sweeps) and, at every POSITIVE call,
    check the exact-sum fast form against the literal restatement on the same state."""
    g = O.OGraph.from_edges(n, s, d, w)
    calls = 0
    level = 0
    while True:
        m = g.m_w / resolution
        a = O.find_assignment(g, m)
        comm, nc, _ = O.extract_components(a)

        def pos(a, comm, nc):
            r1 = O.positive_correction(g, a, comm, nc, m=m, fast=False)
            r2 = O.positive_correction(g, a, comm, nc, m=m, fast=True)
            np.testing.assert_array_equal(r1[0], r2[0])
            assert r1[1:] == r2[1:]
            return r1
        a, ch, *_ = pos(a, comm, nc)
        calls += 1
        if ch:
            comm, nc, _ = O.extract_components(a)
        for sw in range(sweeps):
            a, improved, applied, _, _ = O.maximal_correction(g, a, comm, nc, seed, accept_prob,
                                                              level, sw, m)
            if applied:
                comm, nc, _ = O.extract_components(a)
            if not improved:
                break
            a, ch, *_ = pos(a, comm, nc)
            calls += 1
            if ch:
                comm, nc, _ = O.extract_components(a)
        if nc == g.n or level >= 3:
            return calls
        g = O.aggregate(g, comm)
        level += 1


def test_positive_fast_matches_literal(oracle, golden):
    import workloads as W
    cases = []
    for key in _cases(golden):
        n, s, d, w = case_edges(golden, key)
        if np.all(w == np.floor(w)):
            cases.append((n, s, d, w))
    cases += [W.rmat(10, 16, 0, 2), W.rmat(10, 8, 1, 4), W.rgg(3000, 8.0, 3),
              W.dcsbm(n=3000, k=20, size_lo=50, size_hi=300, seed=1), W.generate("c1_sbm")]
    rng = np.random.default_rng(77)
    for t in range(30):
        n = int(rng.integers(5, 300))
        k = int(rng.integers(n, 8 * n))
        s = rng.integers(0, n, k)
        d = rng.integers(0, n, k)
        keep = s != d
        w = rng.integers(1, 5, k).astype(np.float64)
        cases.append((n, s[keep], d[keep], w[keep]))
    calls = 0
    for i, (n, s, d, w) in enumerate(cases):
        for gam in ((1.0, 0.5) if i % 3 == 0 else (1.0,)):
            calls += _loop_compare_positive(oracle, n, s, d, w, seed=i, resolution=gam,
                                            accept_prob=(0.5, 1.0)[i % 2])
    assert calls > 100
