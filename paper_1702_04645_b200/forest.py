"""Assignment forest (forest.py of the reference) backed by the device forest."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = ["AssignmentForest", "extract_components"]


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


_scratch: dict = {}


def _scratch_ctx(n: int) -> _lib.Context:
    """An edgeless n-node device graph used to run extract_components on raw maps."""
    ctx = _scratch.get("ctx")
    if ctx is None:
        ctx = _lib.Context(0)
        _scratch["ctx"] = ctx
        _scratch["n"] = -1
    if _scratch["n"] != n:
        e = np.empty(0, np.int64)
        ctx.build_graph(n, e, e, np.empty(0))
        _scratch["n"] = n
    return ctx


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
