"""Seeded synthetic inputs for the five BASELINE.json configs.

The reference ships none of these generators; they are written here and
documented in DESIGN.md.  Every graph is undirected and fed as two directed edges.
C1/C2 are drawn with numpy's PCG64 on the host; C3-C5 (R-MAT, RGG) use counter-based
hashes evaluated identically on the host and on the GPU (libslm slm_gen_* /
slm_build_rmat / slm_build_rgg), so the bench can generate them in HBM while the oracle
receives the identical edge multiset from the host twin.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib

RMAT_ABC = (0.57, 0.19, 0.19)

CONFIGS = {
    "c1_sbm": dict(kind="sbm", n=1000, blocks=10, p_in=0.10, p_out=0.005, seed=0),
    "c2_dcsbm": dict(kind="dcsbm", n=100_000, k=200, seed=1),
    "c3_rmat22": dict(kind="rmat", scale=22, edge_factor=16, weight_mode=0, seed=2),
    "c4_rgg24": dict(kind="rgg", n=1 << 24, avg_deg=8.0, seed=3),
    "c5_rmat24": dict(kind="rmat", scale=24, edge_factor=32, weight_mode=1, seed=4),
}


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
    """C3 / C5 host twin of the device generator (slm_gen_rmat_host)."""
    n = 1 << scale
    src, dst, w = _lib.gen_rmat_host(scale, edge_factor, *RMAT_ABC, seed, weight_mode)
    return n, src, dst, w


def rgg_radius(n, avg_deg=8.0):
    return math.sqrt(avg_deg / (math.pi * n))


def rgg(n, avg_deg=8.0, seed=0):
    """C4 host twin of the device generator (slm_gen_rgg_host)."""
    src, dst, w = _lib.gen_rgg_host(n, rgg_radius(n, avg_deg), seed)
    return n, src, dst, w


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
    raise KeyError(name)


def build_on_device(ctx: _lib.Context, name, **over):
    """Generate a named config directly in HBM and build it as level 0."""
    spec = dict(CONFIGS[name])
    spec.update(over)
    kind = spec["kind"]
    if kind == "rmat":
        ctx.build_rmat(spec["scale"], spec["edge_factor"], *RMAT_ABC, spec["seed"],
                       spec["weight_mode"])
    elif kind == "rgg":
        ctx.build_rgg(spec["n"], rgg_radius(spec["n"], spec["avg_deg"]), spec["seed"])
    else:
        n, s, d, w = generate(name, **over)
        ctx.build_graph(n, s, d, w)
