"""Assignment forest (forest.py of the reference) backed by the device forest."""

from __future__ import annotations

from dataclasses import dataclass, field

import threading

import numpy as np

from . import _lib

__all__ = ["AssignmentForest", "extract_components", "reverse_assignment"]


@dataclass
class AssignmentForest:
    """Assignment map plus its component structure (forest.py:23-40)."""
    a: np.ndarray
    comm: np.ndarray
    n_comms: int
    on_cycle: np.ndarray
    _members: list | None = field(default=None, repr=False)

    def community_members(self) -> list:
        if self._members is None:
            order = np.argsort(self.comm, kind="stable")
            bounds = np.searchsorted(self.comm[order], np.arange(self.n_comms + 1))
            self._members = [order[bounds[c]:bounds[c + 1]] for c in range(self.n_comms)]
        return self._members


_tls = threading.local()


def _scratch_ctx(n: int) -> _lib.Context:
    """This thread's device context for map-only calls (extract_components on raw maps,
    reverse_assignment, canonicalize_labels, uniform01): an edgeless n-node graph (n = 0:
    any graph; the map-only entry points do not use it)."""
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = _lib.Context(0)
        _tls.ctx = ctx
        _tls.n = -1
    if n > 0 and _tls.n != n:
        e = np.empty(0, np.int64)
        ctx.build_graph(n, e, e, np.empty(0))
        _tls.n = n
    return ctx


def reverse_assignment(a):
    """forest.py:70-80 on the device: CSR (ptr, kids) of the children j != i with a[j] == i,
    ascending per parent (stable radix sort by target)."""
    a = np.asarray(a, dtype=np.int64)
    if a.size == 0:
        return np.zeros(1, np.int64), np.empty(0, np.int64)
    if a.min() < 0 or a.max() >= a.size:
        raise ValueError("assignment out of range")
    return _scratch_ctx(0).reverse_assignment(a)


def extract_components(a) -> AssignmentForest:
    """forest.py:43-67 on the device: WCC of i -> a[i], labels by smallest member."""
    a = np.asarray(a, dtype=np.int64)
    n = a.size
    if n == 0:
        e = np.empty(0, dtype=np.int64)
        return AssignmentForest(a, e, 0, np.empty(0, dtype=bool))
    if a.min() < 0 or a.max() >= n:
        raise ValueError("assignment out of range")
    ctx = _scratch_ctx(n)
    ctx.set_assignment(a)
    _, comm, nc, oc = ctx.forest(want_a=False)
    return AssignmentForest(a.copy(), comm, nc, oc)
