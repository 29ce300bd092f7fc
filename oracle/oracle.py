"""ctypes front-end of the C oracle (oracle/slm_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / ``--impl reference``
leg import this module, and only as the parity checker or the timed CPU baseline.  The
product package (paper_1702_04645_b200) never imports it.

The functions mirror the reference's phase functions one for one and carry the same
semantics (file:line cited on each); ``run`` restates the level loop of
detector.py:548-653 over the C phases.  ``resolution`` is applied the way SURVEY.md
§8(c) pins the oracle: every gain uses m_w / gamma, the reported score is
(intra - gamma * null) / m_w.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libslm_oracle.so")
SRC_PATH = os.path.join(_HERE, "slm_oracle.c")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, OpenMP for the CPU baseline)."""
    if force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        cmd = ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
               "-fopenmp", "-Wall", "-Wno-maybe-uninitialized", "-o", LIB_PATH, SRC_PATH]
        subprocess.check_call(cmd)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        i64 = C.c_int64
        L.orc_graph_new.restype = vp
        L.orc_graph_new.argtypes = [i64, _i64p, _i64p, _f64p, i64]
        L.orc_graph_free.argtypes = [vp]
        L.orc_graph_sizes.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64),
                                      C.POINTER(C.c_double)]
        L.orc_graph_csr.argtypes = [vp, _i64p, _i64p, _f64p]
        L.orc_graph_union.argtypes = [vp, _i64p, _i64p, _f64p]
        L.orc_graph_strengths.argtypes = [vp, _f64p, _f64p]
        L.orc_aggregate.restype = vp
        L.orc_aggregate.argtypes = [vp, _i64p, i64]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_assign.argtypes = [vp, C.c_double, _i64p]
        L.orc_components.restype = i64
        L.orc_components.argtypes = [i64, _i64p, _i64p, _u8p]
        L.orc_aggregates.argtypes = [vp, _i64p, i64, _f64p, _f64p, _i64p]
        L.orc_local_gains.argtypes = [vp, C.c_double, _i64p, i64, _f64p]
        L.orc_positive.restype = C.c_int
        L.orc_positive.argtypes = [vp, C.c_double, _i64p, _i64p, i64, i64,
                                   C.POINTER(i64), C.POINTER(i64), _f64p, i64, C.POINTER(i64)]
        L.orc_positive_fast.restype = C.c_int
        L.orc_positive_fast.argtypes = L.orc_positive.argtypes
        L.orc_graph_rows.argtypes = [vp, C.c_int, i64, i64, vp, vp, vp]
        L.orc_graph_integral.restype = C.c_int
        L.orc_graph_integral.argtypes = [vp]
        L.orc_plan.argtypes = [vp, C.c_double, _i64p, i64, _i64p]
        L.orc_plan_rows.argtypes = [vp, C.c_double, _i64p, _f64p, _f64p, i64, i64, _i64p]
        L.orc_plan_sample.argtypes = [_i64p, _i64p, _f64p, _f64p, _f64p, C.c_double, _i64p,
                                      _f64p, _f64p, i64, i64, _i64p]
        L.orc_mix_key.restype = C.c_uint64
        L.orc_mix_key.argtypes = [C.c_uint64, i64, i64]
        L.orc_uniform01.argtypes = [C.c_uint64, i64, i64, _i64p, i64, _f64p]
        L.orc_maximal.restype = C.c_int
        L.orc_maximal.argtypes = [vp, C.c_double, _i64p, _i64p, i64, C.c_uint64, C.c_double,
                                  i64, i64, C.POINTER(i64), _f64p, i64, C.POINTER(i64)]
        L.orc_score.restype = C.c_double
        L.orc_score.argtypes = [vp, _i64p, C.c_double]
        L.orc_pairwise_sum.restype = C.c_double
        L.orc_pairwise_sum.argtypes = [_f64p, i64]
        _lib = L
    return _lib


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


class OGraph:
    """Canonical directed CSR + neighbour union + strengths (graph.py:63-175, 257-263)."""

    def __init__(self, handle):
        self._h = handle
        n, ne, ue, m = C.c_int64(), C.c_int64(), C.c_int64(), C.c_double()
        lib().orc_graph_sizes(handle, C.byref(n), C.byref(ne), C.byref(ue), C.byref(m))
        self.n, self.ne, self.ue, self.m_w = n.value, ne.value, ue.value, m.value
        self.integral = bool(lib().orc_graph_integral(handle))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_graph_free(self._h)
            self._h = None

    @classmethod
    def from_edges(cls, n, src, dst, w) -> "OGraph":
        """Graph.from_edges (graph.py:84-116) including its ValueError checks (90-96)."""
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
        return cls(lib().orc_graph_new(n, src, dst, w, src.size))

    def csr(self):
        p = np.empty(self.n + 1, np.int64)
        d = np.empty(self.ne, np.int64)
        w = np.empty(self.ne, np.float64)
        lib().orc_graph_csr(self._h, p, d, w)
        return p, d, w

    def union(self):
        p = np.empty(self.n + 1, np.int64)
        d = np.empty(self.ue, np.int64)
        u = np.empty(self.ue, np.float64)
        lib().orc_graph_union(self._h, p, d, u)
        return p, d, u

    def rows(self, which, r0, r1):
        """rows [r0, r1) of the CSR (which = 0) or the union (which = 1)."""
        p = np.empty(r1 - r0 + 1, np.int64)
        lib().orc_graph_rows(self._h, which, r0, r1, p.ctypes.data, None, None)
        d = np.empty(int(p[-1]), np.int64)
        w = np.empty(int(p[-1]), np.float64)
        lib().orc_graph_rows(self._h, which, r0, r1, p.ctypes.data, d.ctypes.data, w.ctypes.data)
        return p, d, w

    def strengths(self):
        so = np.empty(self.n, np.float64)
        si = np.empty(self.n, np.float64)
        lib().orc_graph_strengths(self._h, so, si)
        return so, si, self.m_w


def _i64(x):
    return np.ascontiguousarray(x, dtype=np.int64)


def find_assignment(g: OGraph, m=None) -> np.ndarray:
    """detector.py:149-158."""
    a = np.empty(g.n, np.int64)
    lib().orc_assign(g._h, g.m_w if m is None else m, a)
    return a


def extract_components(a):
    """forest.py:43-67 -> (comm, n_comms, on_cycle)."""
    a = _i64(a)
    comm = np.empty(a.size, np.int64)
    oc = np.empty(a.size, np.uint8)
    nc = lib().orc_components(a.size, a, comm, oc)
    return comm, int(nc), oc.astype(bool)


def aggregates(g: OGraph, labels, n_comms):
    so = np.empty(max(n_comms, 1), np.float64)
    si = np.empty(max(n_comms, 1), np.float64)
    cnt = np.empty(max(n_comms, 1), np.int64)
    lib().orc_aggregates(g._h, _i64(labels), n_comms, so, si, cnt)
    return so[:n_comms], si[:n_comms], cnt[:n_comms]


def local_gains(g: OGraph, labels, n_comms, m=None):
    """quality.py:170-183."""
    lg = np.empty(g.n, np.float64)
    lib().orc_local_gains(g._h, g.m_w if m is None else m, _i64(labels), n_comms, lg)
    return lg


def positive_correction(g: OGraph, a, comm, n_comms, scc_cut_cap=10_000, m=None, fast=None):
    """detector.py:338-362 -> (a_new, changed, splits, unresolved, gains, n_warnings).

    ``fast`` (default: whenever the graph's weights are integers) selects the exact-sum
    evaluation order of orc_positive_fast -- the same outputs, O(part) per cut instead of a
    subtree search per member (slm_oracle.c); ``fast=False`` forces the literal form."""
    a = _i64(a).copy()
    splits, unres, nw = C.c_int64(), C.c_int64(), C.c_int64()
    cap = g.n + 1
    gains = np.empty(cap, np.float64)
    if fast is None:
        fast = g.integral
    if fast and not g.integral:
        raise ValueError("the fast POSITIVE form needs integer weights")
    fn = lib().orc_positive_fast if fast else lib().orc_positive
    ch = fn(g._h, g.m_w if m is None else m, a, _i64(comm), n_comms,
                            scc_cut_cap, C.byref(splits), C.byref(unres), gains, cap,
                            C.byref(nw))
    return a, bool(ch), splits.value, unres.value, list(gains[:min(splits.value, cap)]), nw.value


def best_targets(g: OGraph, labels, n_comms, m=None):
    """_best_targets over all rows (detector.py:367-418)."""
    cstar = np.empty(g.n, np.int64)
    lib().orc_plan(g._h, g.m_w if m is None else m, _i64(labels), n_comms, cstar)
    return cstar


def plan_sample(uptr, unbr, uu, s_out, s_in, m, labels, S_out, S_in, r0, r1):
    """_best_targets for rows [r0, r1) from raw arrays (uptr relative to r0); returns cstar
    for those rows (bench CPU baseline, all threads set by set_threads)."""
    n = labels.size
    cstar = np.zeros(n, np.int64)
    lib().orc_plan_sample(_i64(uptr), _i64(unbr), np.ascontiguousarray(uu, np.float64),
                          np.ascontiguousarray(s_out, np.float64),
                          np.ascontiguousarray(s_in, np.float64), float(m), _i64(labels),
                          np.ascontiguousarray(S_out, np.float64),
                          np.ascontiguousarray(S_in, np.float64), int(r0), int(r1), cstar)
    return cstar[r0:r1]


def mix_key(seed, level, sweep):
    return int(lib().orc_mix_key(seed & ((1 << 64) - 1), level, sweep))


def uniform01(seed, level, sweep, ids):
    """rng.py:34-43 with parts = (level, sweep)."""
    ids = _i64(ids)
    out = np.empty(ids.size, np.float64)
    lib().orc_uniform01(seed & ((1 << 64) - 1), level, sweep, ids, ids.size, out)
    return out


def maximal_correction(g: OGraph, a, comm, n_comms, seed, accept_prob, level, sweep, m=None):
    """detector.py:457-521 -> (a_new, improved, applied, gains, n_candidates)."""
    a = _i64(a).copy()
    applied, ncand = C.c_int64(), C.c_int64()
    cap = g.n + 1
    gains = np.empty(cap, np.float64)
    imp = lib().orc_maximal(g._h, g.m_w if m is None else m, a, _i64(comm), n_comms,
                            seed & ((1 << 64) - 1), accept_prob, level, sweep,
                            C.byref(applied), gains, cap, C.byref(ncand))
    return a, bool(imp), applied.value, list(gains[:applied.value]), ncand.value


def aggregate(g: OGraph, labels) -> OGraph:
    """graph.py:266-280 (dense-label ValueError included)."""
    labels = _i64(labels)
    if labels.shape != (g.n,):
        raise ValueError("labels must cover every node exactly once")
    c = int(labels.max()) + 1
    if labels.min() < 0 or np.bincount(labels, minlength=c).min() == 0:
        raise ValueError("labels must be a dense relabeling 0..c-1")
    return OGraph(lib().orc_aggregate(g._h, labels, c))


def score(g: OGraph, labels, resolution=1.0) -> float:
    """quality.py:104-118 (modularity; resolution scales the null term)."""
    return float(lib().orc_score(g._h, _i64(labels), float(resolution)))


def pairwise_sum(x) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib().orc_pairwise_sum(x, x.size))


@dataclass
class OracleResult:
    levels: list
    flat: np.ndarray
    final_score: float
    sweeps_per_level: list
    accepted_moves: int = 0
    accepted_splits: int = 0
    unresolved_negative: int = 0
    warnings: list = field(default_factory=list)


def run(n, src, dst, w, seed=0, accept_prob=0.5, max_outer_iters=100,
        scc_cut_cap=10_000, resolution=1.0, graph: OGraph | None = None) -> OracleResult:
    """The level loop of detector.py:548-653 over the C phases."""
    g0 = graph if graph is not None else OGraph.from_edges(n, src, dst, w)
    if g0.n == 0:
        raise ValueError("graph has no nodes")
    g = g0
    levels = []
    res = OracleResult([], None, 0.0, [])
    level = 0
    while True:
        m = g.m_w / resolution
        a = find_assignment(g, m)
        comm, nc, _ = extract_components(a)
        a, ch, sp, un, _, nw = positive_correction(g, a, comm, nc, scc_cut_cap, m)
        if ch:
            comm, nc, _ = extract_components(a)
        res.accepted_splits += sp
        res.unresolved_negative += un
        sweeps = 0
        while True:
            if sweeps >= max_outer_iters:
                res.warnings.append(f"level {level}: stopped after {max_outer_iters} sweeps")
                break
            a, improved, applied, _, _ = maximal_correction(
                g, a, comm, nc, seed, accept_prob, level, sweeps, m)
            if applied:
                comm, nc, _ = extract_components(a)
            sweeps += 1
            res.accepted_moves += applied
            if not improved:
                break
            a, ch, sp, un, _, nw = positive_correction(g, a, comm, nc, scc_cut_cap, m)
            if ch:
                comm, nc, _ = extract_components(a)
            res.accepted_splits += sp
            res.unresolved_negative += un
        res.sweeps_per_level.append(sweeps)
        levels.append(comm)
        if nc == g.n:
            break
        g = aggregate(g, comm)
        level += 1
    flat = levels[0]
    for lv in levels[1:]:
        flat = lv[flat]
    res.levels = levels
    res.flat = flat
    res.final_score = score(g0, flat, resolution)
    return res
