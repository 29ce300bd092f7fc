"""Modularity and gain kernels (quality.py of the reference) on the device."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .graph import Graph, Strengths

__all__ = ["CommunityAggregates", "community_aggregates", "local_gains", "score"]


@dataclass
class CommunityAggregates:
    """Per-community strength sums and member counts (quality.py:52-79)."""
    s_out: np.ndarray
    s_in: np.ndarray
    count: np.ndarray

    @property
    def n_comms(self) -> int:
        return int(self.count.shape[0])


def _load_labels(graph: Graph, labels):
    labels = np.asarray(labels, dtype=np.int64)
    if labels.shape != (graph.n,):
        raise ValueError("labels must cover every node exactly once")
    ctx = graph.context()
    ctx.plan(comm=labels)   # loads the snapshot labels + device aggregates
    return ctx, int(labels.max()) + 1 if labels.size else 0


def community_aggregates(graph: Graph, labels) -> CommunityAggregates:
    """CommunityAggregates.from_labels (quality.py:71-79) computed on the device."""
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
