"""GPU parity: the sm_100a path (through the C ABI) against the reference's golden vectors
and the C oracle.

Bar: bit-exact partitions, assignment maps, candidate targets, sweep counts and statistics
for integer / dyadic weights (all sums exact); final modularity within 1e-12 relative.
The canonical CSR, union, strengths, m_w and ASSIGN are bit-exact for real weights too
(their summation orders are replicated); for real weights the later phases are checked
against a tolerance (NMI >= 0.999, |dQ| <= 1e-9), since their group sums use atomics.
"""

import numpy as np
import pytest

from tests.conftest import case_edges, case_names, exact_sums

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slm():
    import paper_1702_04645_b200 as P
    from paper_1702_04645_b200 import _lib
    _lib.load()
    return P


def nmi(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    n = a.size
    _, ia = np.unique(a, return_inverse=True)
    _, ib = np.unique(b, return_inverse=True)
    cont = np.zeros((ia.max() + 1, ib.max() + 1))
    np.add.at(cont, (ia, ib), 1)
    pa = cont.sum(1) / n
    pb = cont.sum(0) / n
    pab = cont / n
    nz = pab > 0
    mi = (pab[nz] * np.log(pab[nz] / np.outer(pa, pb)[nz])).sum()
    ha = -(pa[pa > 0] * np.log(pa[pa > 0])).sum()
    hb = -(pb[pb > 0] * np.log(pb[pb > 0])).sum()
    return 1.0 if ha + hb == 0 else 2 * mi / (ha + hb)


def test_build_matches_reference_bit_exact(slm, golden):
    for key in case_names(golden):
        n, s, d, w = case_edges(golden, key)
        ctx = slm.Graph.from_edges(n, s, d, w).context()
        p, dst, ww = ctx.csr()
        np.testing.assert_array_equal(p, golden[f"{key}/out_ptr"], err_msg=key)
        np.testing.assert_array_equal(dst, golden[f"{key}/out_dst"], err_msg=key)
        np.testing.assert_array_equal(ww, golden[f"{key}/out_w"], err_msg=key)
        up, un, uu = ctx.union()
        np.testing.assert_array_equal(up, golden[f"{key}/uptr"], err_msg=key)
        np.testing.assert_array_equal(un, golden[f"{key}/unbr"], err_msg=key)
        np.testing.assert_array_equal(uu, golden[f"{key}/uu"], err_msg=key)
        so, si, m = ctx.strengths()
        np.testing.assert_array_equal(so, golden[f"{key}/s_out"], err_msg=key)
        np.testing.assert_array_equal(si, golden[f"{key}/s_in"], err_msg=key)
        assert m == float(golden[f"{key}/m_w"]), key


def test_assign_components_bit_exact(slm, golden):
    for key in case_names(golden):
        n, s, d, w = case_edges(golden, key)
        g = slm.Graph.from_edges(n, s, d, w)
        a = slm.find_assignment(g)
        np.testing.assert_array_equal(a, golden[f"{key}/assign"], err_msg=key)
        f = slm.extract_components(a)
        np.testing.assert_array_equal(f.comm, golden[f"{key}/comm0"], err_msg=key)
        np.testing.assert_array_equal(f.on_cycle, golden[f"{key}/on_cycle0"], err_msg=key)


def test_local_gains_and_plan(slm, golden):
    for key in case_names(golden):
        n, s, d, w = case_edges(golden, key)
        g = slm.Graph.from_edges(n, s, d, w)
        lg = slm.local_gains(g, None, golden[f"{key}/comm0"])
        ref = golden[f"{key}/lg0"]
        if exact_sums(key):
            np.testing.assert_array_equal(lg, ref, err_msg=key)
        else:
            np.testing.assert_allclose(lg, ref, rtol=0, atol=1e-12)
        cstar = g.context().plan(golden[f"{key}/pos_comm"])
        np.testing.assert_array_equal(cstar, golden[f"{key}/cstar"], err_msg=key)


def test_positive_and_maximal_phases(slm, golden):
    for key in case_names(golden):
        if not exact_sums(key):
            continue
        n, s, d, w = case_edges(golden, key)
        seed, p = int(golden[f"{key}/seed"]), float(golden[f"{key}/p"])
        g = slm.Graph.from_edges(n, s, d, w)
        cfg = slm.RunConfig(seed=seed, accept_prob=p)
        f = slm.extract_components(golden[f"{key}/assign"])
        f2, sp, un, gains = slm.positive_correction(g, None, f, cfg)
        np.testing.assert_array_equal(f2.a, golden[f"{key}/pos_a"], err_msg=key)
        np.testing.assert_array_equal(f2.comm, golden[f"{key}/pos_comm"], err_msg=key)
        assert [sp, un] == list(golden[f"{key}/pos_stats"]), key
        np.testing.assert_array_equal(gains, golden[f"{key}/pos_gains"], err_msg=key)
        f3, imp, app, g3 = slm.maximal_correction(g, None, f2, cfg, 0, 0)
        np.testing.assert_array_equal(f3.a, golden[f"{key}/max_a"], err_msg=key)
        np.testing.assert_array_equal(f3.comm, golden[f"{key}/max_comm"], err_msg=key)
        assert [int(imp), app] == list(golden[f"{key}/max_stats"]), key
        np.testing.assert_array_equal(g3, golden[f"{key}/max_gains"], err_msg=key)


def test_full_runs_golden(slm, golden):
    for key in case_names(golden):
        n, s, d, w = case_edges(golden, key)
        seed, p = int(golden[f"{key}/seed"]), float(golden[f"{key}/p"])
        r = slm.run(slm.Graph.from_edges(n, s, d, w), slm.RunConfig(seed=seed, accept_prob=p))
        q = float(golden[f"{key}/final_score"])
        if exact_sums(key):
            assert len(r.hierarchy.levels) == int(golden[f"{key}/nlevels"]), key
            for t, lv in enumerate(r.hierarchy.levels):
                np.testing.assert_array_equal(lv, golden[f"{key}/level{t}"], err_msg=key)
            assert r.stats.sweeps_per_level == list(golden[f"{key}/sweeps"]), key
            assert [r.stats.accepted_moves, r.stats.accepted_splits,
                    r.stats.unresolved_negative] == list(golden[f"{key}/run_stats"]), key
            assert abs(r.final_score - q) <= 1e-12 * max(1.0, abs(q)), key
        else:
            assert nmi(r.hierarchy.flat, golden[f"{key}/flat"]) >= 0.999 or \
                abs(r.final_score - q) <= 1e-9, key


def test_config_fixtures_full_runs(slm, golden_configs):
    import workloads as GN
    G = golden_configs
    specs = {"c1_sbm": lambda: GN.generate("c1_sbm"),
             "c2_dcsbm_small": lambda: GN.dcsbm(n=3000, k=20, size_lo=50, size_hi=300, seed=1),
             "c3_rmat10": lambda: GN.rmat(10, 16, 0, 2),
             "c4_rgg4096": lambda: GN.rgg(4096, 8.0, 3),
             "c5_rmat10w": lambda: GN.rmat(10, 8, 1, 4)}
    for key, fn in specs.items():
        n, s, d, w = fn()
        r = slm.run(slm.Graph.from_edges(n, s, d, w), slm.RunConfig(seed=0))
        assert len(r.hierarchy.levels) == int(G[f"{key}/nlevels"]), key
        for t, lv in enumerate(r.hierarchy.levels):
            np.testing.assert_array_equal(lv, G[f"{key}/level{t}"], err_msg=key)
        assert r.stats.sweeps_per_level == list(G[f"{key}/sweeps"]), key
        assert [r.stats.accepted_moves, r.stats.accepted_splits, r.stats.unresolved_negative] \
            == list(G[f"{key}/run_stats"]), key
        q = float(G[f"{key}/final_score"])
        assert abs(r.final_score - q) <= 1e-12 * abs(q), key


def _vs_oracle(slm, oracle, n, s, d, w, seed=0, p=0.5, gamma=1.0):
    r = slm.run(slm.Graph.from_edges(n, s, d, w),
                slm.RunConfig(seed=seed, accept_prob=p, resolution=gamma))
    o = oracle.run(n, s, d, w, seed=seed, accept_prob=p, resolution=gamma)
    assert len(r.hierarchy.levels) == len(o.levels)
    for x, y in zip(r.hierarchy.levels, o.levels):
        np.testing.assert_array_equal(x, y)
    assert r.stats.sweeps_per_level == o.sweeps_per_level
    assert [r.stats.accepted_moves, r.stats.accepted_splits, r.stats.unresolved_negative] == \
        [o.accepted_moves, o.accepted_splits, o.unresolved_negative]
    assert abs(r.final_score - o.final_score) <= 1e-12 * max(1.0, abs(o.final_score))
    return r


def test_scaled_configs_vs_oracle(slm, oracle):
    import workloads as GN
    oracle.set_threads(8)
    cases = [GN.rmat(13, 16, 0, 2), GN.rmat(13, 16, 1, 4), GN.rgg(1 << 14, 8.0, 3),
             GN.dcsbm(n=20_000, k=60, size_lo=100, size_hi=1000, seed=1)]
    for n, s, d, w in cases:
        _vs_oracle(slm, oracle, n, s, d, w)


def test_resolution_vs_oracle(slm, oracle):
    import workloads as GN
    n, s, d, w = GN.rmat(12, 8, 1, 4)
    for gamma in (0.5, 2.0):
        _vs_oracle(slm, oracle, n, s, d, w, gamma=gamma)
    n, s, d, w = GN.generate("c1_sbm")
    for gamma in (0.5, 2.0):
        _vs_oracle(slm, oracle, n, s, d, w, gamma=gamma)


def test_accept_prob_and_seeds_vs_oracle(slm, oracle):
    import workloads as GN
    n, s, d, w = GN.rmat(11, 16, 1, 7)
    for seed, p in ((3, 1.0), (5, 0.25), (9, 0.75)):
        _vs_oracle(slm, oracle, n, s, d, w, seed=seed, p=p)


def test_kats(slm):
    tri = [(0, 1, 1.0), (1, 2, 1.0), (2, 0, 1.0), (3, 4, 1.0), (4, 5, 1.0), (5, 3, 1.0)]
    s, d, w = (np.array(x) for x in zip(*tri))
    g = slm.Graph.from_edges(6, s, d, w)
    np.testing.assert_array_equal(slm.find_assignment(g), [1, 0, 0, 4, 3, 3])
    assert slm.score(g, None, [0, 0, 0, 1, 1, 1]) == 0.5
    r = slm.run(g, slm.RunConfig(accept_prob=1.0))
    assert [lv.tolist() for lv in r.hierarchy.levels] == [[0, 0, 0, 1, 1, 1], [0, 1]]
    assert r.final_score == 0.5
    r = slm.run(slm.Graph.from_edges(2, [0], [1], [1.0]))
    np.testing.assert_array_equal(r.hierarchy.flat, [0, 1])
    assert len(r.hierarchy.levels) == 1
    # isolated nodes and self-loops only
    r = slm.run(slm.Graph.from_edges(4, [0, 2], [0, 2], [1.0, 2.0]))
    np.testing.assert_array_equal(r.hierarchy.flat, [0, 1, 2, 3])
    # edgeless graph: identity, score 0
    r = slm.run(slm.Graph.from_edges(3, np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0)))
    np.testing.assert_array_equal(r.hierarchy.flat, [0, 1, 2])
    assert r.final_score == 0.0


def test_components_random_functional_graphs(slm):
    """Arbitrary maps (cycles of any length) take the general pointer-doubling path."""
    rng = np.random.default_rng(3)
    from oracle import oracle as O
    for _ in range(40):
        n = int(rng.integers(1, 300))
        a = rng.integers(0, n, size=n).astype(np.int64)
        f = slm.extract_components(a)
        comm, nc, oc = O.extract_components(a)
        np.testing.assert_array_equal(f.comm, comm)
        np.testing.assert_array_equal(f.on_cycle, oc)
        assert f.n_comms == nc


def test_uniform01_device(slm, golden):
    ids = golden["rng/ids"]
    np.testing.assert_array_equal(slm.uniform01(0, (0, 0), ids), golden["rng/u_0_0_0"])
    np.testing.assert_array_equal(slm.uniform01(11, (2, 5), ids), golden["rng/u_11_2_5"])


def test_device_generators_match_host(slm):
    import workloads as W
    from paper_1702_04645_b200 import _lib, generators as GN
    for name, over in (("c3_rmat22", dict(scale=12)), ("c5_rmat24", dict(scale=12, edge_factor=8)),
                       ("c4_rgg24", dict(n=1 << 13))):
        ctx_d = _lib.Context(0)
        GN.build_on_device(ctx_d, {**W.CONFIGS[name], **over})
        n, s, d, w = W.generate(name, **over)
        ctx_h = _lib.Context(0)
        ctx_h.build_graph(n, s, d, w)
        for x, y in zip(ctx_d.csr(), ctx_h.csr()):
            np.testing.assert_array_equal(x, y)


def test_giant_part_executor_parity(slm, golden, oracle, monkeypatch):
    """Force the incremental grid executor (normally for parts > 4096 members) onto every
    bad community and check the same bit-exact outcomes."""
    import workloads as GN
    monkeypatch.setenv("SLM_SMALL_PART", "3")
    for key in case_names(golden):
        if not exact_sums(key):
            continue
        n, s, d, w = case_edges(golden, key)
        seed, p = int(golden[f"{key}/seed"]), float(golden[f"{key}/p"])
        g = slm.Graph.from_edges(n, s, d, w)
        cfg = slm.RunConfig(seed=seed, accept_prob=p)
        f = slm.extract_components(golden[f"{key}/assign"])
        f2, sp, un, gains = slm.positive_correction(g, None, f, cfg)
        np.testing.assert_array_equal(f2.a, golden[f"{key}/pos_a"], err_msg=key)
        assert [sp, un] == list(golden[f"{key}/pos_stats"]), key
        np.testing.assert_array_equal(gains, golden[f"{key}/pos_gains"], err_msg=key)
    for n, s, d, w in (GN.rmat(12, 16, 1, 4), GN.generate("c1_sbm")):
        _vs_oracle(slm, oracle, n, s, d, w)
    monkeypatch.setenv("SLM_SMALL_PART", "64")
    n, s, d, w = GN.rmat(13, 16, 1, 5)
    _vs_oracle(slm, oracle, n, s, d, w)


def test_positive_large_rmat_vs_oracle(slm, oracle):
    """Hub communities well beyond the warp executor (R-MAT 16): one POSITIVE call."""
    import workloads as GN
    n, s, d, w = GN.rmat(16, 16, 1, 4)
    g = slm.Graph.from_edges(n, s, d, w)
    a = slm.find_assignment(g)
    f = slm.extract_components(a)
    f2, sp, un, gains = slm.positive_correction(g, None, f, slm.RunConfig())
    og = oracle.OGraph.from_edges(n, s, d, w)
    comm, nc, _ = oracle.extract_components(a)
    a2, ch, osp, oun, ogains, _ = oracle.positive_correction(og, a, comm, nc)
    np.testing.assert_array_equal(f2.a, a2)
    assert (sp, un) == (osp, oun)
    np.testing.assert_array_equal(gains, ogains)


def _hub_graph(seed=7):
    """Random weighted graph whose rows fill every degree bin, hubs included (rows of
    20k-70k entries span several hub segments)."""
    rng = np.random.default_rng(seed)
    n = 120_000
    src = [rng.integers(0, n, 400_000)]
    dst = [rng.integers(0, n, 400_000)]
    for h, k in enumerate([70_000, 45_000, 30_000, 21_000, 17_000, 12_000, 6_000, 2_500,
                           900, 300, 100, 40]):
        nb = rng.choice(n, size=k, replace=False)
        src.append(np.full(k, h * 997 + 5))
        dst.append(nb)
    s = np.concatenate(src)
    d = np.concatenate(dst)
    keep = s != d
    s, d = s[keep], d[keep]
    w = rng.integers(1, 101, s.size).astype(np.float64)
    return n, np.concatenate([s, d]), np.concatenate([d, s]), np.concatenate([w, w])


def test_plan_all_degree_bins_vs_oracle(slm, oracle):
    """Plan sweep over rows of every degree bin (warp, CTA and hub kernels) against the
    oracle's _best_targets; repeated sweeps check that the tables are left empty."""
    n, s, d, w = _hub_graph()
    ctx = slm.Graph.from_edges(n, s, d, w).context()
    og = oracle.OGraph.from_edges(n, s, d, w)
    rng = np.random.default_rng(11)
    for labels in (rng.integers(0, 2000, n), np.arange(n) // 7, rng.integers(0, 40, n)):
        _, inv = np.unique(labels, return_inverse=True)
        labels = inv.astype(np.int64)
        ref = oracle.best_targets(og, labels, int(labels.max()) + 1)
        for _ in range(2):   # repeated sweeps reuse the emptied tables
            np.testing.assert_array_equal(ctx.plan(labels), ref)


def test_aggregate_long_runs_real_weights_bit_exact(slm, oracle):
    """Coarse edges merging >4096 duplicates (the batched long-run path) keep numpy's
    reduceat order bit for bit, with real-valued weights."""
    rng = np.random.default_rng(5)
    n = 20_000
    s = rng.integers(0, n, 300_000)
    d = rng.integers(0, n, 300_000)
    keep = s != d
    s, d = s[keep], d[keep]
    w = rng.random(s.size) * 3.0 + 0.01
    labels = (np.arange(n) * 7 // n).astype(np.int64)   # 7 dense communities
    g = slm.Graph.from_edges(n, s, d, w)
    ga = slm.aggregate(g, labels)
    og = oracle.aggregate(oracle.OGraph.from_edges(n, s, d, w), labels)
    p, dst, ww = ga.context().csr()
    op, odst, oww = og.csr()
    np.testing.assert_array_equal(p, op)
    np.testing.assert_array_equal(dst, odst)
    np.testing.assert_array_equal(ww, oww)


def test_heavy_member_routing_parity(slm, oracle, monkeypatch):
    """Communities holding a member whose union row exceeds SLM_HEAVY_DEG entries go to the
    CTA executor even when they are small in members (coarse-level hubs).  Force the routing
    with a tiny threshold and compare the whole hierarchy with the oracle."""
    import workloads as GN
    monkeypatch.setenv("SLM_HEAVY_DEG", "24")
    for n, s, d, w in (GN.rmat(13, 16, 1, 6), GN.generate("c1_sbm")):
        _vs_oracle(slm, oracle, n, s, d, w)


def test_plan_without_sweep_view_matches(slm, tmp_path):
    """The integer sweep over the degree-ordered view (default) and over the level graph
    itself (SLM_VIEW=0, read once per process) give identical targets."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "plan.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {root!r})\n"
        "import paper_1702_04645_b200 as slm\n"
        "from tests.test_gpu_parity import _hub_graph\n"
        "n, s, d, w = _hub_graph()\n"
        "ctx = slm.Graph.from_edges(n, s, d, w).context()\n"
        "rng = np.random.default_rng(3)\n"
        "out = [ctx.plan(rng.integers(0, k, n).astype(np.int64)) for k in (30, 3000, n // 5)]\n"
        "np.save(sys.argv[1], np.stack(out))\n")
    res = {}
    for view in ("1", "0"):
        env = dict(os.environ, SLM_VIEW=view)
        f = tmp_path / f"out{view}.npy"
        subprocess.run([sys.executable, str(script), str(f)], check=True, env=env, cwd=root)
        res[view] = np.load(f)
    np.testing.assert_array_equal(res["1"], res["0"])


def test_cta_walkers_full_run_parity(tmp_path):
    """Commit walkers over long timelines use a whole CTA (SLM_WALK_LONG events, read once
    per process): force them onto short timelines and compare full hierarchies with the
    oracle in a subprocess."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "walk.py"
    script.write_text(
        "import sys\n"
        f"sys.path.insert(0, {root!r})\n"
        "import paper_1702_04645_b200 as slm\n"
        "import workloads as GN\n"
        "from oracle import oracle as O\n"
        "from tests.test_gpu_parity import _vs_oracle\n"
        "O.build()\n"
        "for n, s, d, w in (GN.rmat(13, 16, 1, 4), GN.rmat(12, 16, 0, 2), GN.generate('c1_sbm')):\n"
        "    _vs_oracle(slm, O, n, s, d, w)\n"
        "print('ok')\n")
    env = dict(os.environ, SLM_WALK_LONG="40")
    r = subprocess.run([sys.executable, str(script)], env=env, cwd=root, capture_output=True,
                       text=True)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_big_candidate_items_parity(slm, oracle, monkeypatch):
    """Commit candidates whose tails hold many entries are priced by work items spread over
    the GPU (integer weights: exact fp64 atomics).  Force every candidate with more than 8
    tail entries onto that path and compare whole hierarchies with the oracle."""
    import workloads as GN
    monkeypatch.setenv("SLM_BIG_VOL", "8")
    for n, s, d, w in (GN.rmat(13, 16, 1, 4), GN.rmat(12, 16, 0, 7), GN.generate("c1_sbm")):
        _vs_oracle(slm, oracle, n, s, d, w)


def test_local_gains_without_wown_matches(tmp_path):
    """POSITIVE's local gains from the sweep's own-community sums (kept across commits by
    deltas; default) and from a full pass over the union (SLM_WOWN=0) give the same
    hierarchies."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "wown.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {root!r})\n"
        "import paper_1702_04645_b200 as slm\n"
        "import workloads as GN\n"
        "out = []\n"
        "for n, s, d, w in (GN.rmat(14, 16, 1, 4), GN.rgg(1 << 14, 8.0, 3)):\n"
        "    r = slm.run(slm.Graph.from_edges(n, s, d, w), slm.RunConfig())\n"
        "    out += list(r.hierarchy.levels) + [np.array(r.stats.sweeps_per_level),\n"
        "            np.array([r.stats.accepted_moves, r.stats.accepted_splits, r.stats.unresolved_negative])]\n"
        "np.savez(sys.argv[1], *out)\n")
    res = {}
    for mode in ("1", "0"):
        f = tmp_path / f"w{mode}.npz"
        subprocess.run([sys.executable, str(script), str(f)], check=True, cwd=root,
                       env=dict(os.environ, SLM_WOWN=mode))
        res[mode] = np.load(f)
    assert res["1"].files == res["0"].files
    for k in res["1"].files:
        np.testing.assert_array_equal(res["1"][k], res["0"][k])


@pytest.mark.gpu
def test_walker_runs_match_single_commits(tmp_path):
    """Commit walkers deciding the simple events after a commit in one pass (default) and
    one event per step (SLM_WALK_RUNS=0) give the same hierarchies, at gamma 1 and 0.5."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "runs.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {root!r})\n"
        "import paper_1702_04645_b200 as slm\n"
        "import workloads as GN\n"
        "out = []\n"
        "for (n, s, d, w), gam in ((GN.rmat(15, 16, 1, 4), 1.0), (GN.rmat(15, 16, 1, 4), 0.5),\n"
        "                          (GN.generate('c1_sbm'), 0.5)):\n"
        "    r = slm.run(slm.Graph.from_edges(n, s, d, w), slm.RunConfig(resolution=gam))\n"
        "    out += list(r.hierarchy.levels) + [np.array(r.stats.sweeps_per_level),\n"
        "            np.array([r.stats.accepted_moves, r.stats.accepted_splits, r.stats.unresolved_negative]),\n"
        "            np.array([r.final_score])]\n"
        "np.savez(sys.argv[1], *out)\n")
    res = {}
    for mode in ("1", "0"):
        f = tmp_path / f"r{mode}.npz"
        subprocess.run([sys.executable, str(script), str(f)], check=True, cwd=root,
                       env=dict(os.environ, SLM_WALK_RUNS=mode))
        res[mode] = np.load(f)
    assert res["1"].files == res["0"].files
    for k in res["1"].files:
        np.testing.assert_array_equal(res["1"][k], res["0"][k])
