"""Graph container with the reference's construction semantics (graph.py).

``Graph.from_edges`` validates exactly like the reference (graph.py:84-96, ValueError on
mismatched lengths, out-of-range ids or non-positive / non-finite weights) and keeps the
edge list; the canonical CSR, the neighbour union and the strengths are built on the GPU
(libslm ``slm_build_graph``: device radix sort + run merge, graph.py:97-116 and 151-175)
the first time the graph is used, and stay resident in the graph's device context.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["Graph", "GraphFormatError", "NeighborUnion", "Strengths", "aggregate",
           "canonicalize_labels", "compose_labels", "strengths"]


class GraphFormatError(ValueError):
    """Malformed edge-list or partition input (graph.py:33-34)."""


@dataclass(frozen=True)
class Strengths:
    """Out/in strength per node and the total edge weight m_w (graph.py:37-43)."""
    s_out: np.ndarray
    s_in: np.ndarray
    m_w: float


@dataclass(frozen=True)
class NeighborUnion:
    """Per-node union of out- and in-neighbours, self-loops excluded (graph.py:46-60).

    ``w_out[e] = W(i, j)`` and ``w_in[e] = W(j, i)`` (0.0 when absent) for entry e = (i, j),
    split on the device from the canonical CSR (slm_get_union_split).  Every gain kernel
    consumes only w_out + w_in, which the device stores pre-summed as ``u``;
    ``w_out + w_in == u`` bit for bit.
    """
    ptr: np.ndarray
    nbr: np.ndarray
    row: np.ndarray
    w_out: np.ndarray
    w_in: np.ndarray
    u: np.ndarray


class Graph:
    """Immutable directed weighted graph; dense 0-based node ids (graph.py:63-148)."""

    def __init__(self, n, src, dst, w, _validated=False):
        self.n = int(n)
        self._src = src
        self._dst = dst
        self._w = w
        self._parent = None   # (graph, labels, n_comms) of a graph made by aggregate()
        self._ctx = None
        self._csr = None
        self._union = None
        self._st = None

    @classmethod
    def from_edges(cls, n, src, dst, w) -> "Graph":
        n = int(n)
        src = np.ascontiguousarray(src, dtype=np.int64)
        dst = np.ascontiguousarray(dst, dtype=np.int64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        if not (src.shape == dst.shape == w.shape):
            raise ValueError("src, dst, w must have equal length")
        if src.size:
            if src.min() < 0 or dst.min() < 0 or src.max() >= n or dst.max() >= n:
                raise ValueError("edge endpoint out of range")
            if not np.isfinite(w).all() or (w <= 0).any():
                raise ValueError("edge weights must be finite and positive")
        return cls(n, src, dst, w, _validated=True)

    # --------------------------------------------------------------- device state
    def context(self, level0: bool = True) -> _lib.Context:
        """Device context holding this graph as hierarchy level 0 (built on first use)."""
        if self._ctx is None or (level0 and self._ctx.level != 0):
            if self._ctx is None:
                self._ctx = _lib.Context(0)
            if self._parent is not None:
                parent, labels, c = self._parent
                self._ctx.build_aggregate(parent.context(), labels, c)
            else:
                self._ctx.build_graph(self.n, self._src, self._dst, self._w)
        return self._ctx

    def _canonical(self):
        if self._csr is None:
            p, d, w = self.context().csr()
            for arr in (p, d, w):
                arr.setflags(write=False)
            self._csr = (p, d, w)
        return self._csr

    @property
    def out_ptr(self):
        return self._canonical()[0]

    @property
    def out_dst(self):
        return self._canonical()[1]

    @property
    def out_w(self):
        return self._canonical()[2]

    @property
    def edge_count(self) -> int:
        return int(self.out_dst.shape[0])

    def edge_rows(self) -> np.ndarray:
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.out_ptr))

    def neighbor_union(self) -> NeighborUnion:
        if self._union is None:
            ctx = self.context()
            p, nb, u = ctx.union()
            wo, wi = ctx.union_split()
            row = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(p))
            for arr in (p, nb, row, wo, wi, u):
                arr.setflags(write=False)
            self._union = NeighborUnion(p, nb, row, wo, wi, u)
        return self._union

    def out_slice(self, i):
        lo, hi = self.out_ptr[i], self.out_ptr[i + 1]
        return self.out_dst[lo:hi], self.out_w[lo:hi]

    def __eq__(self, other):
        if not isinstance(other, Graph):
            return NotImplemented
        return self.n == other.n and all(
            np.array_equal(a, b) for a, b in zip(self._canonical(), other._canonical()))

    def __repr__(self):
        return f"Graph(n={self.n}, edges={self.edge_count})"


def strengths(graph: Graph) -> Strengths:
    """graph.py:257-263, computed on the device (sequential per-row sums, pairwise m_w)."""
    if graph._st is None:
        so, si, m = graph.context().strengths()
        so.setflags(write=False)
        si.setflags(write=False)
        graph._st = Strengths(so, si, m)
    return graph._st


def aggregate(graph: Graph, labels) -> Graph:
    """graph.py:266-280: collapse communities into super-nodes.  The coarse graph is built on
    the device from the parent's resident CSR (relabel + the level build's radix sort and
    run merge: slm_build_aggregate); intra-community weight becomes self-loops."""
    labels = np.asarray(labels, dtype=np.int64)
    if labels.shape != (graph.n,):
        raise ValueError("labels must cover every node exactly once")
    if graph.n == 0:
        return Graph.from_edges(0, labels, labels, np.empty(0))
    c = int(labels.max()) + 1
    if labels.min() < 0 or np.bincount(labels, minlength=c).min() == 0:
        raise ValueError("labels must be a dense relabeling 0..c-1")
    out = Graph(c, None, None, None, _validated=True)
    out._parent = (graph, labels.copy(), c)
    out._ctx = _lib.Context(0)
    out._ctx.build_aggregate(graph.context(), labels, c)
    return out


def canonicalize_labels(labels) -> np.ndarray:
    """Dense labels 0..c-1 ordered by each community's smallest member (graph.py:283-291),
    on the device (stable radix sort by label, first occurrences ranked)."""
    labels = np.asarray(labels, dtype=np.int64)
    if labels.size == 0:
        return labels.copy()
    from .forest import _scratch_ctx
    out, _ = _scratch_ctx(0).canonicalize(labels)
    return out


def compose_labels(inner, outer) -> np.ndarray:
    """node -> inner community -> outer community (graph.py:294-298)."""
    return np.asarray(outer, dtype=np.int64)[np.asarray(inner, dtype=np.int64)]
