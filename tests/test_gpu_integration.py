"""The reference-side backend stub of INTEGRATION.md (integration/synclouvain_b200.py) runs
the whole level loop over the C ABI alone and reproduces the reference's golden
hierarchies (tests/golden/reference_phases.npz, exact-sum cases)."""

import os

import numpy as np
import pytest

from tests.conftest import ROOT, case_edges, case_names, exact_sums

pytestmark = pytest.mark.gpu


class _RefGraph:
    """The reference Graph's duck type (n, edge_rows(), out_dst, out_w), from its CSR."""

    def __init__(self, g):
        self.n = g.n
        self.out_ptr, self.out_dst, self.out_w = g.out_ptr, g.out_dst, g.out_w

    def edge_rows(self):
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.out_ptr))


def test_reference_side_stub(golden):
    import importlib.util
    import paper_1702_04645_b200 as P
    spec = importlib.util.spec_from_file_location(
        "synclouvain_b200", os.path.join(ROOT, "integration", "synclouvain_b200.py"))
    stub = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(stub)
    lib = os.path.join(ROOT, "paper_1702_04645_b200", "libslm.so")
    checked = 0
    for key in case_names(golden):
        if not exact_sums(key):
            continue
        n, s, d, w = case_edges(golden, key)
        g = _RefGraph(P.Graph.from_edges(n, s, d, w))
        cfg = P.RunConfig(seed=int(golden[f"{key}/seed"]), accept_prob=float(golden[f"{key}/p"]))
        r = stub.run(g, cfg, lib_path=lib)
        assert len(r.hierarchy.levels) == int(golden[f"{key}/nlevels"])
        for t, lv in enumerate(r.hierarchy.levels):
            np.testing.assert_array_equal(lv, golden[f"{key}/level{t}"])
        np.testing.assert_array_equal(r.hierarchy.flat, golden[f"{key}/flat"])
        assert r.stats.sweeps_per_level == list(golden[f"{key}/sweeps"])
        assert [r.stats.accepted_moves, r.stats.accepted_splits, r.stats.unresolved_negative] \
            == list(golden[f"{key}/run_stats"])
        assert abs(r.final_score - float(golden[f"{key}/final_score"])) <= \
            1e-12 * max(1.0, abs(float(golden[f"{key}/final_score"])))
        checked += 1
    assert checked >= 10
