"""Reference-side GPU backend stub: ``synclouvain.run`` over libslm.so's C ABI.

This is the file a synclouvain maintainer would add (e.g. as ``synclouvain/_b200.py``) to
let the reference package dispatch ``run(graph, config)`` (detector.py:548-653) to the B200
library.  It needs only ctypes + numpy and the reference's own Graph / RunConfig objects
(duck-typed: ``graph.n``, ``graph.edge_rows()``, ``graph.out_dst``, ``graph.out_w``;
``config.seed`` / ``accept_prob`` / ``max_outer_iters`` / ``scc_cut_cap``), and returns the
reference's result shape.  It is the complete level loop -- ASSIGN, COMPONENTS, POSITIVE,
{MAXIMAL -> POSITIVE} up to max_outer_iters, AGGREGATE -- with the reference's stop rules
and statistics; tests/test_gpu_integration.py runs it against the golden hierarchies.
"""

from __future__ import annotations

import ctypes as C
import os
from types import SimpleNamespace

import numpy as np

_VP, _I64, _I32, _D = C.c_void_p, C.c_int64, C.c_int32, C.c_double
_PI64, _PI32, _PD = C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_double)


class _Cfg(C.Structure):   # slm_config (include/slm.h)
    _fields_ = [("seed", C.c_uint64), ("accept_prob", C.c_double),
                ("max_outer_iters", C.c_int64), ("scc_cut_cap", C.c_int64),
                ("resolution", C.c_double)]


_SIG = {
    "slm_create": (_VP, [C.c_int]), "slm_destroy": (None, [_VP]),
    "slm_last_error": (C.c_char_p, [_VP]),
    "slm_build_graph": (C.c_int, [_VP, _I64, _VP, _VP, _VP, _I64]),
    "slm_graph_info": (C.c_int, [_VP, _PI64, _PI64, _PI64, _PD, _PI32]),
    "slm_set_resolution": (C.c_int, [_VP, _D]),
    "slm_assign": (C.c_int, [_VP, _VP]),
    "slm_components": (C.c_int, [_VP, _VP, _VP, _PI64]),
    "slm_get_forest": (C.c_int, [_VP, _VP, _VP, _VP, _PI64]),
    "slm_positive": (C.c_int, [_VP, C.POINTER(_Cfg), _PI64, _PI64, _PI32, _VP, _I64]),
    "slm_maximal": (C.c_int, [_VP, C.POINTER(_Cfg), _I64, _I64, _PI32, _PI64, _VP, _I64]),
    "slm_aggregate": (C.c_int, [_VP]),
    "slm_score": (C.c_int, [_VP, _I32, _VP, _D, _PD]),
}


def _load(path=None):
    L = C.CDLL(path or os.environ.get("SLM_LIB", "libslm.so"))
    for name, (res, args) in _SIG.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


def run(graph, config, lib_path=None):
    """synclouvain.run on the GPU -> SimpleNamespace(hierarchy(levels, flat), final_score,
    stats(levels, sweeps_per_level, accepted_moves, accepted_splits, unresolved_negative))."""
    L = _load(lib_path)
    if graph.n == 0:
        raise ValueError("graph has no nodes")
    ctx = L.slm_create(0)
    if not ctx:
        raise RuntimeError("slm_create failed: no usable CUDA device")

    def ok(rc):
        if rc:
            msg = L.slm_last_error(ctx).decode()
            raise (ValueError if rc == -1 else RuntimeError)(msg)

    def p(a):
        return None if a is None else a.ctypes.data_as(C.c_void_p)

    try:
        rows = np.ascontiguousarray(graph.edge_rows(), np.int64)
        dst = np.ascontiguousarray(graph.out_dst, np.int64)
        w = np.ascontiguousarray(graph.out_w, np.float64)
        ok(L.slm_build_graph(ctx, graph.n, p(rows), p(dst), p(w), rows.size))
        cfg = _Cfg(config.seed & ((1 << 64) - 1), float(config.accept_prob),
                   int(config.max_outer_iters), int(config.scc_cut_cap),
                   float(getattr(config, "resolution", 1.0)))
        ok(L.slm_set_resolution(ctx, cfg.resolution))
        stats = SimpleNamespace(levels=0, sweeps_per_level=[], accepted_moves=0,
                                accepted_splits=0, unresolved_negative=0, warnings=[])
        sp, un, app = C.c_int64(), C.c_int64(), C.c_int64()
        ch, imp = C.c_int32(), C.c_int32()
        levels = []
        level = 0
        while True:                                             # detector.py:573
            n, ne, ue, fl = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
            mw = C.c_double()
            ok(L.slm_graph_info(ctx, C.byref(n), C.byref(ne), C.byref(ue), C.byref(mw),
                                C.byref(fl)))
            ok(L.slm_assign(ctx, None))                          # :578
            nc = C.c_int64()
            ok(L.slm_components(ctx, None, None, C.byref(nc)))   # :580
            ok(L.slm_positive(ctx, C.byref(cfg), C.byref(sp), C.byref(un), C.byref(ch),
                              None, 0))                          # :583
            stats.accepted_splits += sp.value
            stats.unresolved_negative += un.value
            sweeps = 0
            while True:                                          # :596-629
                if sweeps >= cfg.max_outer_iters:
                    stats.warnings.append(f"level {level}: stopped after "
                                          f"{cfg.max_outer_iters} sweeps")
                    break
                ok(L.slm_maximal(ctx, C.byref(cfg), level, sweeps, C.byref(imp),
                                 C.byref(app), None, 0))
                sweeps += 1
                stats.accepted_moves += app.value
                if not imp.value:
                    break
                ok(L.slm_positive(ctx, C.byref(cfg), C.byref(sp), C.byref(un), C.byref(ch),
                                  None, 0))
                stats.accepted_splits += sp.value
                stats.unresolved_negative += un.value
            stats.sweeps_per_level.append(sweeps)
            comm = np.empty(n.value, np.int64)
            ok(L.slm_get_forest(ctx, None, p(comm), None, C.byref(nc)))
            levels.append(comm)                                  # :631-632
            if nc.value == n.value:                              # :636-637
                break
            ok(L.slm_aggregate(ctx))                             # :639-641
            level += 1
        flat = levels[0]
        for lv in levels[1:]:
            flat = lv[flat]                                      # compose_labels
        q = C.c_double()
        ok(L.slm_score(ctx, 1, p(np.ascontiguousarray(flat, np.int64)), cfg.resolution,
                       C.byref(q)))
        stats.levels = len(levels)
        return SimpleNamespace(hierarchy=SimpleNamespace(levels=levels, flat=flat),
                               final_score=q.value, stats=stats)
    finally:
        L.slm_destroy(ctx)
