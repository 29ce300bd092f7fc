"""Seeded synthetic inputs for the five BASELINE.json configs (DESIGN.md §6 "Synthetic inputs").

Input generation only -- neither the product nor the oracle.  The reference ships none of
these generators; every graph is undirected and fed as two directed edges.

* C1 / C2 (SBM, DC-SBM) are drawn with numpy's PCG64 on the host.
* C3-C5 (R-MAT, RGG) are counter-based hashes (``gen_host.c``, compiled into
  ``libslm_gen.so`` with OpenMP).  The product's device generators (``slm_build_rmat`` /
  ``slm_build_rgg`` in libslm.so) draw the identical edge multiset in HBM;
  tests/test_gpu_parity.py checks the device CSR against the one built from these edges.

Nothing here loads libslm.so, so the ``bench.py --impl reference`` arm and the oracle get
their inputs without touching the product library.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libslm_gen.so")
SRC_PATH = os.path.join(_HERE, "gen_host.c")

RMAT_ABC = (0.57, 0.19, 0.19)

CONFIGS = {
    "c1_sbm": dict(kind="sbm", n=1000, blocks=10, p_in=0.10, p_out=0.005, seed=0),
    "c2_dcsbm": dict(kind="dcsbm", n=100_000, k=200, seed=1),
    "c3_rmat22": dict(kind="rmat", scale=22, edge_factor=16, weight_mode=0, seed=2),
    "c4_rgg24": dict(kind="rgg", n=1 << 24, avg_deg=8.0, seed=3),
    "c5_rmat24": dict(kind="rmat", scale=24, edge_factor=32, weight_mode=1, seed=4),
    # device-generated pair-model twins of C1 / C2 (counter hashes instead of numpy's PCG64)
    "c1_sbm_hash": dict(kind="sbm_hash", n=1000, blocks=10, p_in=0.10, p_out=0.005, seed=0),
    "c2_dcsbm_hash": dict(kind="dcsbm_hash", n=100_000, k=200, seed=1),
}


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-Wall",
                               "-o", LIB_PATH, SRC_PATH])
    return LIB_PATH


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.gen_rmat.restype = C.c_int64
        L.gen_rmat.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                               C.c_uint64, C.c_int, vp, vp, vp]
        L.gen_pairs.restype = C.c_int64
        L.gen_pairs.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_double, vp, vp,
                                vp, vp, C.c_double, C.c_uint64, vp, vp, vp]
        L.gen_rgg.restype = C.c_int64
        L.gen_rgg.argtypes = [C.c_int64, C.c_double, C.c_uint64, vp, vp, vp]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _sym(n, s, d, w=None):
    s = np.asarray(s, np.int64)
    d = np.asarray(d, np.int64)
    if w is None:
        w = np.ones(s.size, np.float64)
    return n, np.concatenate([s, d]), np.concatenate([d, s]), np.concatenate([w, w])


def sbm(n=1000, blocks=10, p_in=0.10, p_out=0.005, seed=0):
    """C1: planted partition, blocks of n/blocks consecutive ids, Bernoulli per pair i<j."""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, k=1)
    bs = n // blocks
    p = np.where(iu // bs == ju // bs, p_in, p_out)
    keep = rng.random(iu.size) < p
    return _sym(n, iu[keep], ju[keep])


def _powerlaw(rng, size, lo, hi, exp):
    u = rng.random(size)
    if abs(exp - 1.0) < 1e-12:
        return lo * (hi / lo) ** u
    a, b = lo ** (1.0 - exp), hi ** (1.0 - exp)
    return (a + u * (b - a)) ** (1.0 / (1.0 - exp))


def dcsbm(n=100_000, k=200, size_lo=100, size_hi=1000, size_exp=1.0, deg_lo=5.0, deg_hi=200.0,
          deg_exp=2.5, mu=0.3, seed=1):
    """C2: degree-corrected SBM with Chung-Lu edges.

    Community sizes ~ x^-size_exp on [size_lo, size_hi], renormalised to sum to n; expected
    degrees theta ~ x^-deg_exp on [deg_lo, deg_hi]; a fraction mu of every node's expected
    degree goes to other communities.  Intra-community pairs are Bernoulli with
    p = min(1, k_i k_j / K_c) (k = (1-mu) theta, K_c = sum over the community); inter-
    community edges are Chung-Lu with weights mu*theta (Poisson(O/2) endpoint pairs drawn
    proportionally to the weights, same-community pairs rejected).  Node ids are permuted.
    Symmetrised, deduplicated, unit weights.
    """
    rng = np.random.default_rng(seed)
    raw = _powerlaw(rng, k, size_lo, size_hi, size_exp)
    exact = raw / raw.sum() * n
    sizes = np.floor(exact).astype(np.int64)
    rem = n - int(sizes.sum())
    sizes[np.argsort(-(exact - sizes), kind="stable")[:rem]] += 1
    perm = rng.permutation(n)
    comm_of = np.empty(n, np.int64)
    comm_of[perm] = np.repeat(np.arange(k), sizes)
    theta = _powerlaw(rng, n, deg_lo, deg_hi, deg_exp)
    kin = (1.0 - mu) * theta
    kout = mu * theta
    src, dst = [], []
    starts = np.concatenate([[0], np.cumsum(sizes)])
    for c in range(k):
        mem = perm[starts[c]:starts[c + 1]]
        kk = kin[mem]
        K = kk.sum()
        iu, ju = np.triu_indices(mem.size, k=1)
        p = np.minimum(1.0, kk[iu] * kk[ju] / K)
        keep = rng.random(iu.size) < p
        src.append(mem[iu[keep]])
        dst.append(mem[ju[keep]])
    O = kout.sum()
    m_out = rng.poisson(O / 2.0)
    prob = kout / O
    a = rng.choice(n, size=m_out, p=prob)
    b = rng.choice(n, size=m_out, p=prob)
    ok = comm_of[a] != comm_of[b]
    src.append(a[ok])
    dst.append(b[ok])
    s = np.concatenate(src)
    d = np.concatenate(dst)
    lo, hi = np.minimum(s, d), np.maximum(s, d)
    key = np.unique(lo * n + hi)
    return _sym(n, key // n, key % n)


def rmat(scale, edge_factor, weight_mode=0, seed=0):
    """C3 / C5: R-MAT (a, b, c) = RMAT_ABC, ids permuted, self-loops dropped, both directions
    of every draw (duplicates are merged by the graph build); weights 1 or U[1, 100]."""
    L = _L()
    n = 1 << scale
    k = L.gen_rmat(scale, edge_factor, *RMAT_ABC, seed, weight_mode, None, None, None)
    src = np.empty(k, np.int64)
    dst = np.empty(k, np.int64)
    w = np.empty(k, np.float64)
    L.gen_rmat(scale, edge_factor, *RMAT_ABC, seed, weight_mode, _p(src), _p(dst), _p(w))
    return n, src, dst, w


def rgg_radius(n, avg_deg=8.0):
    return math.sqrt(avg_deg / (math.pi * n))


def rgg(n, avg_deg=8.0, seed=0):
    """C4: random geometric graph in the unit square, r = sqrt(avg_deg / (pi n))."""
    L = _L()
    r = rgg_radius(n, avg_deg)
    k = L.gen_rgg(n, r, seed, None, None, None)
    src = np.empty(k, np.int64)
    dst = np.empty(k, np.int64)
    w = np.empty(k, np.float64)
    L.gen_rgg(n, r, seed, _p(src), _p(dst), _p(w))
    return n, src, dst, w


def dcsbm_params(n=100_000, k=200, size_lo=100, size_hi=1000, size_exp=1.0, deg_lo=5.0,
                 deg_hi=200.0, deg_exp=2.5, mu=0.3, seed=1):
    """Per-node parameters of the pair-model DC-SBM (C2's shape): community of every node
    (consecutive blocks of power-law sizes renormalised to n), kin = (1-mu) theta,
    kout = mu theta (theta power law on [deg_lo, deg_hi]), K per community, O."""
    rng = np.random.default_rng(seed)
    raw = _powerlaw(rng, k, size_lo, size_hi, size_exp)
    exact = raw / raw.sum() * n
    sizes = np.floor(exact).astype(np.int64)
    sizes[np.argsort(-(exact - sizes), kind="stable")[:n - int(sizes.sum())]] += 1
    comm = np.repeat(np.arange(k, dtype=np.int32), sizes)
    theta = _powerlaw(rng, n, deg_lo, deg_hi, deg_exp)
    kin = (1.0 - mu) * theta
    kout = mu * theta
    K = np.bincount(comm, weights=kin, minlength=k)
    return comm, kin, kout, K, float(kout.sum())


def _pairs(mode, n, blocks, p_in, p_out, params, seed):
    L = _L()
    comm, kin, kout, K, O = params if params is not None else (None,) * 4 + (1.0,)
    arrs = [None if a is None else np.ascontiguousarray(a) for a in (comm, kin, kout, K)]
    ptrs = [None if a is None else _p(a) for a in arrs]
    k = L.gen_pairs(mode, n, blocks, p_in, p_out, *ptrs, O, seed, None, None, None)
    src = np.empty(k, np.int64)
    dst = np.empty(k, np.int64)
    w = np.empty(k, np.float64)
    L.gen_pairs(mode, n, blocks, p_in, p_out, *ptrs, O, seed, _p(src), _p(dst), _p(w))
    return n, src, dst, w


def sbm_hash(n=1000, blocks=10, p_in=0.10, p_out=0.005, seed=0):
    """Counter-hash planted partition (host twin of the device generator slm_build_pairs)."""
    return _pairs(0, n, blocks, p_in, p_out, None, seed)


def dcsbm_hash(seed=1, **kw):
    """Counter-hash DC-SBM over dcsbm_params (host twin of slm_build_pairs, mode 1)."""
    params = dcsbm_params(seed=seed, **kw)
    return _pairs(1, params[0].size, 0, 0.0, 0.0, params, seed)


def generate(name, **over):
    """Host edge list (n, src, dst, w) of a named config (overrides allowed)."""
    spec = dict(CONFIGS[name])
    spec.update(over)
    kind = spec.pop("kind")
    if kind == "sbm":
        return sbm(**spec)
    if kind == "dcsbm":
        return dcsbm(**spec)
    if kind == "rmat":
        return rmat(spec["scale"], spec["edge_factor"], spec["weight_mode"], spec["seed"])
    if kind == "rgg":
        return rgg(spec["n"], spec["avg_deg"], spec["seed"])
    if kind == "sbm_hash":
        return sbm_hash(**spec)
    if kind == "dcsbm_hash":
        return dcsbm_hash(**spec)
    raise KeyError(name)
