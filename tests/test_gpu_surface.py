"""The rest of the reference's hot-path API surface on the device, bit for bit against the
unmodified reference (tests/golden/reference_surface.npz, make_golden.py --surface):
NeighborUnion.w_out / w_in, reverse_assignment, canonicalize_labels,
CommunityAggregates.from_labels / move_nodes / check, gain_switch and aggregate() -- real-
valued (dyadic and uniform) weights included, since every sum keeps the reference's order."""

import os

import numpy as np
import pytest

from tests.conftest import GOLDEN, case_edges, case_names

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def surf():
    return np.load(os.path.join(GOLDEN, "reference_surface.npz"))


@pytest.fixture(scope="module")
def P():
    import paper_1702_04645_b200 as P
    return P


def test_union_split(P, golden, surf):
    for key in case_names(golden):
        n, s, d, w = case_edges(golden, key)
        U = P.Graph.from_edges(n, s, d, w).neighbor_union()
        np.testing.assert_array_equal(U.w_out, surf[f"{key}/w_out"])
        np.testing.assert_array_equal(U.w_in, surf[f"{key}/w_in"])
        np.testing.assert_array_equal(U.w_out + U.w_in, U.u)


def test_reverse_assignment(P, golden, surf):
    for key in case_names(golden):
        for tag in ("assign", "pos_a", "max_a"):
            p, kids = P.reverse_assignment(golden[f"{key}/{tag}"])
            np.testing.assert_array_equal(p, surf[f"{key}/rev_{tag}_ptr"])
            np.testing.assert_array_equal(kids, surf[f"{key}/rev_{tag}_kids"])


def test_canonicalize_labels(P, golden, surf):
    np.testing.assert_array_equal(P.canonicalize_labels([5, 3, 5, 9, 3]), [0, 1, 0, 2, 1])
    for key in case_names(golden):
        np.testing.assert_array_equal(P.canonicalize_labels(surf[f"{key}/canon_in"]),
                                      surf[f"{key}/canon_out"])
    big = np.random.default_rng(1).integers(0, 1 << 20, 3_000_000)
    uniq, first = np.unique(big, return_index=True)
    remap = np.empty(uniq.size, np.int64)
    remap[np.argsort(first, kind="stable")] = np.arange(uniq.size)
    np.testing.assert_array_equal(P.canonicalize_labels(big), remap[np.searchsorted(uniq, big)])


def test_aggregates_and_gain_switch(P, golden, surf):
    for key in case_names(golden):
        n, s, d, w = case_edges(golden, key)
        g = P.Graph.from_edges(n, s, d, w)
        st = P.strengths(g)
        comm = golden[f"{key}/pos_comm"]
        agg = P.CommunityAggregates.from_labels(st, comm, int(comm.max()) + 1)
        np.testing.assert_array_equal(agg.s_out, surf[f"{key}/agg_s_out"])
        np.testing.assert_array_equal(agg.s_in, surf[f"{key}/agg_s_in"])
        np.testing.assert_array_equal(agg.count, surf[f"{key}/agg_count"])
        assert agg.check(st, comm)
        for t, (frm, to, k, gv) in enumerate(surf[f"{key}/gs"]):
            nodes = surf[f"{key}/gs{t}_nodes"]
            got = P.gain_switch(g, st, comm, agg, nodes, int(frm), None if to < 0 else int(to))
            assert got == gv, (key, t, got, gv)
        # move_nodes keeps the aggregates consistent with the relabeled partition
        frm = int(comm[0])
        mem = np.flatnonzero(comm == frm)[:1]
        to = int(comm.max())
        if to != frm:
            agg.move_nodes(st, mem, frm, to)
            lab = comm.copy()
            lab[mem] = to
            assert agg.check(st, lab)


def test_aggregate_on_device(P, golden, surf):
    for key in case_names(golden):
        n, s, d, w = case_edges(golden, key)
        g = P.Graph.from_edges(n, s, d, w)
        h = P.aggregate(g, golden[f"{key}/pos_comm"])
        np.testing.assert_array_equal(h.out_ptr, surf[f"{key}/agg_graph_ptr"])
        np.testing.assert_array_equal(h.out_dst, surf[f"{key}/agg_graph_dst"])
        np.testing.assert_array_equal(h.out_w, surf[f"{key}/agg_graph_w"])
        # the aggregated graph is a full Graph: run() works on it and rebuilds after use
        r1 = P.run(h, P.RunConfig(seed=1))
        r2 = P.run(h, P.RunConfig(seed=1))
        assert len(r1.hierarchy.levels) == len(r2.hierarchy.levels)
        np.testing.assert_array_equal(r1.hierarchy.flat, r2.hierarchy.flat)
    with pytest.raises(ValueError):
        P.aggregate(g, np.zeros(g.n, np.int64) + 1)
