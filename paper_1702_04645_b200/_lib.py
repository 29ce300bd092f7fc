"""ctypes binding of libslm.so (include/slm.h).

The CUDA library is the only compute path: importing the package does not require a GPU,
but every compute call raises ``RuntimeError`` when the library or a CUDA device is
missing -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SLM_LIB_PATH") or os.path.join(_HERE, "libslm.so")   # (override: A/B runs)

SLM_OK, SLM_EINVAL, SLM_ECUDA, SLM_ENOMEM, SLM_ESTATE, SLM_EUNSUP = 0, -1, -2, -3, -4, -5

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


class SlmConfig(C.Structure):
    """slm_config (include/slm.h): RunConfig (detector.py:22-40) + resolution."""
    _fields_ = [("seed", C.c_uint64), ("accept_prob", C.c_double),
                ("max_outer_iters", C.c_int64), ("scc_cut_cap", C.c_int64),
                ("resolution", C.c_double)]


# every symbol declared in include/slm.h, with its ctypes signature
_VP = C.c_void_p
_I64 = C.c_int64
_PI64 = C.POINTER(C.c_int64)
_PI32 = C.POINTER(C.c_int32)
_PD = C.POINTER(C.c_double)
_NULLABLE_I64 = _PI64
SIGNATURES = {
    "slm_create": (_VP, [C.c_int]),
    "slm_destroy": (None, [_VP]),
    "slm_last_error": (C.c_char_p, [_VP]),
    "slm_stream": (_VP, [_VP]),
    "slm_sync": (C.c_int, [_VP]),
    "slm_build_graph": (C.c_int, [_VP, _I64, _VP, _VP, _VP, _I64]),
    "slm_build_graph_device": (C.c_int, [_VP, _I64, _VP, _VP, _VP, _I64]),
    "slm_graph_info": (C.c_int, [_VP, _PI64, _PI64, _PI64, _PD, _PI32]),
    "slm_get_csr": (C.c_int, [_VP, _VP, _VP, _VP]),
    "slm_get_union": (C.c_int, [_VP, _VP, _VP, _VP]),
    "slm_get_strengths": (C.c_int, [_VP, _VP, _VP]),
    "slm_get_union_rows": (C.c_int, [_VP, _I64, _I64, _VP, _VP, _VP]),
    "slm_get_csr_rows": (C.c_int, [_VP, _I64, _I64, _VP, _VP, _VP]),
    "slm_set_resolution": (C.c_int, [_VP, C.c_double]),
    "slm_assign": (C.c_int, [_VP, _VP]),
    "slm_set_assignment": (C.c_int, [_VP, _VP]),
    "slm_components": (C.c_int, [_VP, _VP, _VP, _PI64]),
    "slm_get_forest": (C.c_int, [_VP, _VP, _VP, _VP, _PI64]),
    "slm_get_aggregates": (C.c_int, [_VP, _VP, _VP, _VP]),
    "slm_local_gains": (C.c_int, [_VP, _VP]),
    "slm_positive": (C.c_int, [_VP, C.POINTER(SlmConfig), _PI64, _PI64, _PI32, _VP, _I64]),
    "slm_plan_sweep": (C.c_int, [_VP, _VP, _VP]),
    "slm_maximal": (C.c_int, [_VP, C.POINTER(SlmConfig), _I64, _I64, _PI32, _PI64, _VP, _I64]),
    "slm_aggregate": (C.c_int, [_VP]),
    "slm_score": (C.c_int, [_VP, C.c_int32, _VP, C.c_double, _PD]),
    "slm_uniform01": (C.c_int, [_VP, C.c_uint64, _I64, _I64, _VP, _I64, _VP]),
    "slm_last_commit_stats": (C.c_int, [_VP, _PI64, _PI64]),
    "slm_phase_times": (C.c_int, [_VP, _VP, C.c_int32, C.c_int32]),
    "slm_plan_sweep_async": (C.c_int, [_VP, C.c_int32]),
    "slm_plan_groups": (C.c_int, [_VP, _PI64, _VP, _VP]),
    "slm_get_cstar": (C.c_int, [_VP, _VP]),
    "slm_debug_sweep_floor": (C.c_int, [_VP, C.c_int32, _PD]),
    "slm_run": (C.c_int, [_VP, C.POINTER(SlmConfig), _PI64, _VP, _VP]),
    "slm_run_level": (C.c_int, [_VP, _I64, _PI64, _PI64, _PI32, _VP]),
    "slm_community_sums": (C.c_int, [_VP, _I64, _VP, _I64, _VP, _VP, _VP, _VP, _VP]),
    "slm_gain_switch": (C.c_int, [_VP, _VP, _VP, _I64, _I64, _I64, _VP, C.c_double, _PD]),
    "slm_reverse_assignment": (C.c_int, [_VP, _I64, _VP, _VP, _VP, _PI64]),
    "slm_get_union_split": (C.c_int, [_VP, _VP, _VP]),
    "slm_canonicalize_labels": (C.c_int, [_VP, _I64, _VP, _VP, _PI64]),
    "slm_build_aggregate": (C.c_int, [_VP, _VP, _VP, _I64]),
    "slm_debug_sort": (C.c_int, [_VP, C.c_int32, _VP, _VP, _I64, C.c_int32, _PD]),
    "slm_debug_scan": (C.c_int, [_VP, C.c_int32, _VP, _VP, _VP, _I64]),
    "slm_build_rmat": (C.c_int, [_VP, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                 C.c_uint64, C.c_int]),
    "slm_build_rgg": (C.c_int, [_VP, _I64, C.c_double, C.c_uint64]),
    "slm_build_pairs": (C.c_int, [_VP, C.c_int32, _I64, _I64, C.c_double, C.c_double, _VP, _VP,
                                  _VP, _VP, _I64, C.c_double, C.c_uint64]),
}

_lib = None


def load():
    """Load libslm.so (raises if it has not been built: no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libslm.so not built ({LIB_PATH}); run "
                               "`python -m paper_1702_04645_b200._build`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("SLM_LIB_PATH") and not hasattr(L, name):
                continue   # A/B runs against an older build: its missing entries stay unbound
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def i64(x):
    return np.ascontiguousarray(x, dtype=np.int64)


def f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


class Context:
    """Owns one slm_ctx (one device stream, resident level graph + forest)."""

    def __init__(self, device: int = 0):
        L = load()
        h = L.slm_create(int(device))
        if not h:
            raise RuntimeError("slm_create failed: no usable CUDA device "
                               "(the SLM path has no CPU fallback)")
        self._h = h
        self._L = L
        self.level = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.slm_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def check(self, rc):
        if rc == SLM_OK:
            return
        msg = self._L.slm_last_error(self._h).decode(errors="replace")
        if rc == SLM_EINVAL:
            raise ValueError(msg)
        raise RuntimeError(f"libslm error {rc}: {msg}")

    def call(self, name, *args):
        self.check(getattr(self._L, name)(self._h, *args))

    def stream_ptr(self) -> int:
        return int(self._L.slm_stream(self._h) or 0)

    # ----- graph
    def build_graph(self, n, src, dst, w):
        src, dst, w = i64(src), i64(dst), f64(w)
        self.call("slm_build_graph", int(n), ptr(src), ptr(dst), ptr(w), int(src.size))
        self.level = 0

    def build_rmat(self, scale, edge_factor, a, b, c, seed, weight_mode):
        self.call("slm_build_rmat", int(scale), int(edge_factor), float(a), float(b), float(c),
                  int(seed), int(weight_mode))
        self.level = 0

    def build_rgg(self, n, radius, seed):
        self.call("slm_build_rgg", int(n), float(radius), int(seed))
        self.level = 0

    def build_pairs(self, mode, n, blocks=0, p_in=0.0, p_out=0.0, params=None, seed=0):
        if params is None:
            comm = kin = kout = K = None
            O, nc = 1.0, 0
        else:
            comm, kin, kout, K, O = params
            comm = np.ascontiguousarray(comm, np.int32)
            kin, kout, K = f64(kin), f64(kout), f64(K)
            nc = K.size
        self.call("slm_build_pairs", int(mode), int(n), int(blocks), float(p_in), float(p_out),
                  ptr(comm), ptr(kin), ptr(kout), ptr(K), int(nc), float(O), int(seed))
        self.level = 0

    def info(self):
        n, ne, ue = C.c_int64(), C.c_int64(), C.c_int64()
        m = C.c_double()
        fl = C.c_int32()
        self.call("slm_graph_info", C.byref(n), C.byref(ne), C.byref(ue), C.byref(m), C.byref(fl))
        return dict(n=n.value, ne=ne.value, ue=ue.value, m_w=m.value,
                    symmetric=bool(fl.value & 1), integral=bool(fl.value & 2),
                    plan_path=("u32" if fl.value & 4 else
                               "fp64-exact" if (fl.value & 2) and not (fl.value & 8)
                               else "sorted"))

    def csr(self):
        d = self.info()
        p = np.empty(d["n"] + 1, np.int64)
        dst = np.empty(d["ne"], np.int64)
        w = np.empty(d["ne"], np.float64)
        self.call("slm_get_csr", ptr(p), ptr(dst), ptr(w))
        return p, dst, w

    def union(self):
        d = self.info()
        p = np.empty(d["n"] + 1, np.int64)
        nb = np.empty(d["ue"], np.int64)
        u = np.empty(d["ue"], np.float64)
        self.call("slm_get_union", ptr(p), ptr(nb), ptr(u))
        return p, nb, u

    def union_rows(self, r0, r1):
        p = np.empty(r1 - r0 + 1, np.int64)
        self.call("slm_get_union_rows", int(r0), int(r1), ptr(p), None, None)
        nb = np.empty(int(p[-1]), np.int64)
        u = np.empty(int(p[-1]), np.float64)
        self.call("slm_get_union_rows", int(r0), int(r1), ptr(p), ptr(nb), ptr(u))
        return p, nb, u

    def csr_rows(self, r0, r1):
        p = np.empty(r1 - r0 + 1, np.int64)
        self.call("slm_get_csr_rows", int(r0), int(r1), ptr(p), None, None)
        d = np.empty(int(p[-1]), np.int64)
        w = np.empty(int(p[-1]), np.float64)
        self.call("slm_get_csr_rows", int(r0), int(r1), ptr(p), ptr(d), ptr(w))
        return p, d, w

    def strengths(self):
        d = self.info()
        so = np.empty(d["n"], np.float64)
        si = np.empty(d["n"], np.float64)
        self.call("slm_get_strengths", ptr(so), ptr(si))
        return so, si, d["m_w"]

    def set_resolution(self, gamma):
        self.call("slm_set_resolution", float(gamma))

    # ----- phases
    def assign(self, want=True):
        n = self.info()["n"]
        a = np.empty(n, np.int64) if want else None
        self.call("slm_assign", ptr(a))
        return a

    def set_assignment(self, a):
        a = i64(a)
        self.call("slm_set_assignment", ptr(a))

    def components(self, want=True):
        n = self.info()["n"]
        comm = np.empty(n, np.int64) if want else None
        oc = np.empty(n, np.uint8) if want else None
        nc = C.c_int64()
        self.call("slm_components", ptr(comm), ptr(oc), C.byref(nc))
        return comm, nc.value, (oc.astype(bool) if want else None)

    def forest(self, want_a=True, want_comm=True, want_cycle=True):
        n = self.info()["n"]
        a = np.empty(n, np.int64) if want_a else None
        comm = np.empty(n, np.int64) if want_comm else None
        oc = np.empty(n, np.uint8) if want_cycle else None
        nc = C.c_int64()
        self.call("slm_get_forest", ptr(a), ptr(comm), ptr(oc), C.byref(nc))
        return a, comm, nc.value, (oc.astype(bool) if want_cycle else None)

    def aggregates(self, n_comms):
        so = np.empty(n_comms, np.float64)
        si = np.empty(n_comms, np.float64)
        cnt = np.empty(n_comms, np.int64)
        self.call("slm_get_aggregates", ptr(so), ptr(si), ptr(cnt))
        return so, si, cnt

    def local_gains(self):
        lg = np.empty(self.info()["n"], np.float64)
        self.call("slm_local_gains", ptr(lg))
        return lg

    def positive(self, cfg: SlmConfig, want_gains=False):
        sp, un = C.c_int64(), C.c_int64()
        ch = C.c_int32()
        cap = self.info()["n"] + 1 if want_gains else 0
        g = np.empty(cap, np.float64) if want_gains else None
        self.call("slm_positive", C.byref(cfg), C.byref(sp), C.byref(un), C.byref(ch), ptr(g), cap)
        gains = list(g[:min(sp.value, cap)]) if want_gains else []
        return bool(ch.value), sp.value, un.value, gains

    def plan(self, comm=None):
        n = self.info()["n"]
        cstar = np.empty(n, np.int64)
        self.call("slm_plan_sweep", ptr(None if comm is None else i64(comm)), ptr(cstar))
        return cstar

    def maximal(self, cfg: SlmConfig, level, sweep, want_gains=False):
        imp = C.c_int32()
        app = C.c_int64()
        cap = self.info()["n"] + 1 if want_gains else 0
        g = np.empty(cap, np.float64) if want_gains else None
        self.call("slm_maximal", C.byref(cfg), int(level), int(sweep), C.byref(imp), C.byref(app),
                  ptr(g), cap)
        gains = list(g[:app.value]) if want_gains else []
        return bool(imp.value), app.value, gains

    def aggregate(self):
        self.call("slm_aggregate")
        self.level += 1

    def score(self, labels, gamma=1.0, on_original=True):
        labels = i64(labels)
        q = C.c_double()
        self.call("slm_score", 1 if on_original else 0, ptr(labels), float(gamma), C.byref(q))
        return q.value

    def uniform01(self, seed, level, sweep, ids):
        ids = i64(ids)
        out = np.empty(ids.size, np.float64)
        self.call("slm_uniform01", int(seed) & ((1 << 64) - 1), int(level), int(sweep), ptr(ids),
                  ids.size, ptr(out))
        return out

    def plan_async(self, bin_mask=127):
        self.call("slm_plan_sweep_async", int(bin_mask))

    def plan_groups(self):
        g = C.c_int64()
        rows = np.zeros(6, np.int64)
        ents = np.zeros(6, np.int64)
        self.call("slm_plan_groups", C.byref(g), ptr(rows), ptr(ents))
        return g.value, rows, ents

    def get_cstar(self):
        cstar = np.empty(self.info()["n"], np.int64)
        self.call("slm_get_cstar", ptr(cstar))
        return cstar

    def sweep_floor(self, mode):
        ms = C.c_double()
        self.call("slm_debug_sweep_floor", int(mode), C.byref(ms))
        return ms.value

    def run(self, cfg: SlmConfig):
        """The whole level loop on the device side (slm_run) -> (levels, sweeps, paths,
        capped, stats[5], phase seconds[5])."""
        nl = C.c_int64()
        st = np.zeros(5, np.int64)
        ph = np.zeros(5, np.float64)
        self.call("slm_run", C.byref(cfg), C.byref(nl), ptr(st), ptr(ph))
        levels, sweeps, paths, capped = [], [], [], []
        for t in range(nl.value):
            nn, sw, pp = C.c_int64(), C.c_int64(), C.c_int32()
            self.call("slm_run_level", t, C.byref(nn), C.byref(sw), C.byref(pp), None)
            lab = np.empty(nn.value, np.int64)
            self.call("slm_run_level", t, None, None, None, ptr(lab))
            levels.append(lab)
            sweeps.append(sw.value)
            paths.append(("u32", "fp64-exact", "sorted")[pp.value & 3])
            capped.append(bool(pp.value & 8))
        self.level = nl.value - 1
        return levels, sweeps, paths, capped, st, ph

    # ----- reference API surface (slm_surface.cu)
    def community_sums(self, labels, n_comms, s_out, s_in):
        labels, s_out, s_in = i64(labels), f64(s_out), f64(s_in)
        So = np.empty(n_comms, np.float64)
        Si = np.empty(n_comms, np.float64)
        cnt = np.empty(n_comms, np.int64)
        self.call("slm_community_sums", labels.size, ptr(labels), int(n_comms), ptr(s_out),
                  ptr(s_in), ptr(So), ptr(Si), ptr(cnt))
        return So, Si, cnt

    def gain_switch(self, labels, nodes, frm, to, agg4, m):
        labels, nodes = i64(labels), i64(nodes)
        a4 = f64(agg4)
        g = C.c_double()
        self.call("slm_gain_switch", ptr(labels), ptr(nodes), nodes.size, int(frm),
                  -1 if to is None else int(to), ptr(a4), float(m), C.byref(g))
        return g.value

    def reverse_assignment(self, a):
        a = i64(a)
        p = np.empty(a.size + 1, np.int64)
        kids = np.empty(a.size, np.int64)
        nk = C.c_int64()
        self.call("slm_reverse_assignment", a.size, ptr(a), ptr(p), ptr(kids), C.byref(nk))
        return p, kids[:nk.value].copy()

    def union_split(self):
        ue = self.info()["ue"]
        wo = np.empty(ue, np.float64)
        wi = np.empty(ue, np.float64)
        self.call("slm_get_union_split", ptr(wo), ptr(wi))
        return wo, wi

    def canonicalize(self, labels):
        labels = i64(labels)
        out = np.empty(labels.size, np.int64)
        nc = C.c_int64()
        self.call("slm_canonicalize_labels", labels.size, ptr(labels), ptr(out), C.byref(nc))
        return out, nc.value

    def build_aggregate(self, src: "Context", labels, n_comms):
        labels = i64(labels)
        self.call("slm_build_aggregate", src.handle, ptr(labels), int(n_comms))
        self.level = 0

    def debug_sort(self, keys, vals, end_bit):
        """Stable radix sort of (uint64 keys, f64 vals) or (uint32 keys, int32 vals) by bits
        [0, end_bit) on the device; returns (keys, vals, device ms)."""
        keys = np.ascontiguousarray(keys).copy()
        vals = np.ascontiguousarray(vals).copy()
        kind = 0 if keys.dtype == np.uint64 else 1
        ms = C.c_double()
        self.call("slm_debug_sort", kind, ptr(keys), ptr(vals), keys.size, int(end_bit),
                  C.byref(ms))
        return keys, vals, ms.value

    def debug_scan(self, x, keys=None, out_dtype=None):
        """Exclusive prefix sum on the device (restarting at key changes when keys given)."""
        x = np.ascontiguousarray(x)
        kinds = {(np.int64, np.int64): 0, (np.int32, np.int32): 1, (np.int32, np.int64): 2,
                 (np.float64, np.float64): 3}
        od = np.dtype(out_dtype or x.dtype)
        kind = 4 if keys is not None else kinds[(x.dtype.type, od.type)]
        out = np.empty(x.size, od)
        k = None if keys is None else np.ascontiguousarray(keys, np.uint32)
        self.call("slm_debug_scan", kind, ptr(x), ptr(out), ptr(k), x.size)
        return out

    def sync(self):
        self.call("slm_sync")

    PHASES = ("plan", "candidates", "spec", "walk", "components", "aggregates", "layout",
              "positive_lg", "positive_small", "positive_giant", "assign", "aggregate",
              "alloc_ms", "alloc_calls", "view_build_ms")

    def phase_times(self, reset=False):
        ms = np.zeros(len(self.PHASES), np.float64)
        self.call("slm_phase_times", ptr(ms), len(self.PHASES), 1 if reset else 0)
        return {k: round(float(v), 1) for k, v in zip(self.PHASES, ms)}

    def last_commit_stats(self):
        c, r = C.c_int64(), C.c_int64()
        self.call("slm_last_commit_stats", C.byref(c), C.byref(r))
        return c.value, r.value

