"""Plan-sweep paths other than the integer fast path:
  * the fp64 generic path (integer weights with a row total >= 2^32, e.g. coarse levels of
    C5) -- forced with SLM_FORCE_GENERIC on graphs whose hub rows exceed 4096 entries
    (k_plan_large), bit-exact against the oracle;
  * the sorted reference-order path of real-valued weights (detector.py:383-418 order:
    stable sort by (row, community), reduceat sums) -- bit-exact targets, deterministic
    runs, and full runs past n = 70 within NMI >= 0.999 / |dQ| <= 1e-9 of the oracle."""

import os
import subprocess
import sys

import numpy as np
import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_1702_04645_b200 as slm
import workloads as W
from oracle import oracle as O
O.build()
cases = [W.rmat(16, 16, 1, 4), W.rmat(14, 16, 0, 2), W.generate("c1_sbm")]
for n, s, d, w in cases:
    g = slm.Graph.from_edges(n, s, d, w)
    og = O.OGraph.from_edges(n, s, d, w)
    a = O.find_assignment(og)
    comm, nc, _ = O.extract_components(a)
    a, ch, *_ = O.positive_correction(og, a, comm, nc)
    comm, nc, _ = O.extract_components(a)
    assert np.array_equal(g.context().plan(comm), O.best_targets(og, comm, nc)), "plan"
    r = slm.run(g, slm.RunConfig())
    o = O.run(n, s, d, w)
    assert len(r.hierarchy.levels) == len(o.levels)
    for x, y in zip(r.hierarchy.levels, o.levels):
        assert np.array_equal(x, y), "levels"
    assert r.stats.sweeps_per_level == o.sweeps_per_level
    assert r.stats.plan_paths[0] == {path!r}, r.stats.plan_paths
print("ok")
"""


@pytest.mark.parametrize("env,path", [("SLM_FORCE_GENERIC", "fp64-exact"),
                                      ("SLM_PLAN_SORTED", "sorted")])
def test_forced_paths_vs_oracle(tmp_path, env, path):
    f = tmp_path / "p.py"
    f.write_text(_SCRIPT.format(root=ROOT, path=path))
    r = subprocess.run([sys.executable, str(f)], env=dict(os.environ, **{env: "1"}), cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("env", ["SLM_VIEW_SORTED", "SLM_SOA", "SLM_VIEW"])
def test_integer_sweep_variants_vs_oracle(tmp_path, env):
    """The integer sweep's switches -- view rows in the level graph's entry order instead of
    sorted by view id, {key, sum} slots instead of split tables, no degree-ordered view at
    all -- change the work, never a target or a partition (same checks as the default)."""
    f = tmp_path / "p.py"
    f.write_text(_SCRIPT.format(root=ROOT, path="u32"))
    r = subprocess.run([sys.executable, str(f)], env=dict(os.environ, **{env: "0"}), cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def _real(n, s, d, seed):
    rng = np.random.default_rng(seed)
    w = rng.uniform(0.1, 3.0, s.size)
    return n, s, d, w


def test_real_weights_sorted_path(slm, oracle):
    import workloads as W
    from tests.test_gpu_parity import nmi
    cases = []
    for k, (n, s, d, _) in enumerate([W.rmat(12, 8, 0, 2), W.rgg(1 << 13, 8.0, 3),
                                      W.dcsbm(n=5000, k=30, size_lo=50, size_hi=400, seed=1)]):
        cases.append(_real(n, s, d, k))
    for n, s, d, w in cases:
        g = slm.Graph.from_edges(n, s, d, w)
        og = oracle.OGraph.from_edges(n, s, d, w)
        # targets of the first plan sweep: bit-exact (same order, same fp64 expression)
        a = oracle.find_assignment(og)
        comm, nc, _ = oracle.extract_components(a)
        assert np.array_equal(g.context().plan(comm), oracle.best_targets(og, comm, nc))
        r1 = slm.run(g, slm.RunConfig())
        r2 = slm.run(g, slm.RunConfig())
        assert r1.stats.plan_paths[0] == "sorted"
        for x, y in zip(r1.hierarchy.levels, r2.hierarchy.levels):
            np.testing.assert_array_equal(x, y)      # deterministic
        o = oracle.run(n, s, d, w)
        q_ok = abs(r1.final_score - o.final_score) <= 1e-9
        assert nmi(r1.hierarchy.flat, o.flat) >= 0.999 or q_ok, (n, r1.final_score, o.final_score)


def test_positive_long_cycles_and_scc_cap(slm, oracle):
    """POSITIVE on forests with assignment cycles longer than 2 (only a caller-supplied
    forest has them): the literal executor (slm_positive_lit.cu) against the
    reference's algorithm in the oracle -- branch cuts, pair cuts over the cycle's arcs,
    and the scc_cut_cap peel -- bit for bit, integer and real weights."""
    rng = np.random.default_rng(2024)
    checked = 0
    for t in range(24):
        n = int(rng.integers(6, 60))
        k = int(rng.integers(2 * n, 6 * n))
        s = rng.integers(0, n, k)
        d = rng.integers(0, n, k)
        keep = s != d
        s, d = s[keep], d[keep]
        w = (rng.integers(1, 9, s.size).astype(np.float64) if t % 2 == 0
             else rng.uniform(0.1, 3.0, s.size))
        g = slm.Graph.from_edges(n, s, d, w)
        og = oracle.OGraph.from_edges(n, s, d, w)
        a = rng.integers(0, n, n)          # random functional graph: cycles of any length
        f = slm.extract_components(a)
        comm, nc, _ = oracle.extract_components(a)
        np.testing.assert_array_equal(f.comm, comm)
        for cap in (10_000, 3, 2):
            cfg = slm.RunConfig(scc_cut_cap=cap)
            f2, sp, un, gains = slm.positive_correction(g, None, f, cfg)
            a2, ch, sp2, un2, gains2, _ = oracle.positive_correction(og, a, comm, nc,
                                                                     scc_cut_cap=cap)
            np.testing.assert_array_equal(f2.a, a2)
            assert (sp, un) == (sp2, un2), (t, cap)
            g1, g2 = np.asarray(gains, np.float64), np.asarray(gains2, np.float64)
            if t % 2 == 0:
                np.testing.assert_array_equal(g1, g2)
            else:   # real weights: the <= 2-cycle executors sum in DFS order
                np.testing.assert_allclose(g1, g2, rtol=1e-12, atol=0)
            checked += 1
    assert checked == 72
