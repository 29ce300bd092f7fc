"""Modularity and gain kernels (quality.py of the reference) on the device.

``score``, ``local_gains``, ``gain_switch`` and ``CommunityAggregates.from_labels`` /
``check`` run in libslm (slm_level.cu, slm_lgains.cu, slm_surface.cu) with the reference's
summation orders; ``move_nodes`` / ``remove_node`` are the reference's O(k) scalar updates of
the caller's host arrays (quality.py:81-95), kept on the host like the arrays they mutate.
"""

from __future__ import annotations

import numpy as np

from .graph import Graph, Strengths, strengths

__all__ = ["CommunityAggregates", "community_aggregates", "gain_switch", "local_gains", "score"]


class CommunityAggregates:
    """Per-community strength sums and member counts (quality.py:52-101)."""

    __slots__ = ("s_out", "s_in", "count")

    def __init__(self, s_out, s_in, count):
        self.s_out = s_out
        self.s_in = s_in
        self.count = count

    @property
    def n_comms(self) -> int:
        return int(self.count.shape[0])

    @classmethod
    def from_labels(cls, st: Strengths, labels, n_comms: int | None = None):
        """quality.py:71-79: sequential per-community sums in node order (np.bincount),
        computed on the device (slm_community_sums)."""
        from .forest import _scratch_ctx
        labels = np.asarray(labels, dtype=np.int64)
        if n_comms is None:
            n_comms = int(labels.max()) + 1 if labels.size else 0
        if labels.size and (labels.min() < 0 or labels.max() >= n_comms):
            raise ValueError("labels out of range")
        so, si, cnt = _scratch_ctx(0).community_sums(labels, n_comms, st.s_out, st.s_in)
        return cls(so, si, cnt)

    def remove_node(self, st: Strengths, labels, i: int) -> None:   # quality.py:81-85
        c = int(labels[i])
        self.s_out[c] -= st.s_out[i]
        self.s_in[c] -= st.s_in[i]
        self.count[c] -= 1

    def move_nodes(self, st: Strengths, nodes, frm: int, to: int) -> None:   # quality.py:87-95
        so = st.s_out[nodes].sum()
        si = st.s_in[nodes].sum()
        self.s_out[frm] -= so
        self.s_in[frm] -= si
        self.count[frm] -= len(nodes)
        self.s_out[to] += so
        self.s_in[to] += si
        self.count[to] += len(nodes)

    def check(self, st: Strengths, labels, atol: float = 1e-9) -> bool:   # quality.py:97-101
        fresh = CommunityAggregates.from_labels(st, labels, self.n_comms)
        return (np.array_equal(fresh.count, self.count)
                and np.allclose(fresh.s_out, self.s_out, atol=atol, rtol=0.0)
                and np.allclose(fresh.s_in, self.s_in, atol=atol, rtol=0.0))


def _load_labels(graph: Graph, labels):
    labels = np.asarray(labels, dtype=np.int64)
    if labels.shape != (graph.n,):
        raise ValueError("labels must cover every node exactly once")
    ctx = graph.context()
    ctx.plan(comm=labels)   # loads the snapshot labels + device aggregates
    return ctx, int(labels.max()) + 1 if labels.size else 0


def community_aggregates(graph: Graph, labels) -> CommunityAggregates:
    """CommunityAggregates.from_labels over the graph's own strengths, on the device."""
    ctx, nc = _load_labels(graph, labels)
    so, si, cnt = ctx.aggregates(nc)
    return CommunityAggregates(so, si, cnt)


def score(graph: Graph, st: Strengths | None, labels, params=None, resolution: float = 1.0) -> float:
    """quality.py:104-118: directed modularity (intra - gamma*null)/m_w; 0.0 if edgeless."""
    if params is not None and getattr(params, "model", "modularity") != "modularity":
        raise NotImplementedError("only the modularity model is on the B200 path")
    labels = np.asarray(labels, dtype=np.int64)
    if labels.shape != (graph.n,):
        raise ValueError("labels must cover every node exactly once")
    return graph.context().score(labels, resolution, on_original=True)


def local_gains(graph: Graph, st: Strengths | None, labels, agg=None) -> np.ndarray:
    """quality.py:170-183 on the device (agg is recomputed from labels)."""
    ctx, _ = _load_labels(graph, labels)
    return ctx.local_gains()


def gain_switch(graph: Graph, st: Strengths | None, labels, agg: CommunityAggregates, nodes,
                frm: int, to: int | None, in_set=None) -> float:
    """quality.py:186-219: exact score difference of relabeling ``nodes`` from ``frm`` to
    ``to`` (None: a fresh empty community), on the device over the graph's union rows (per
    row pairwise sums accumulated in node order, the reference's fp64 expression).  The
    moved nodes' strengths are the graph's own; ``st`` supplies m_w (None: the graph's)."""
    if to is not None and to == frm:
        return 0.0
    labels = np.asarray(labels, dtype=np.int64)
    if labels.shape != (graph.n,):
        raise ValueError("labels must cover every node exactly once")
    st = strengths(graph) if st is None else st
    agg4 = [agg.s_out[frm], agg.s_in[frm], 0.0 if to is None else agg.s_out[to],
            0.0 if to is None else agg.s_in[to]]
    return graph.context().gain_switch(labels, np.asarray(nodes, dtype=np.int64), frm, to, agg4,
                                       st.m_w)
