"""Device generation of the BASELINE.json synthetic graphs straight into the level-0 build
(R-MAT, RGG, and the pair-model SBM / DC-SBM twins of C1 / C2).

The counter-based R-MAT (C3, C5) and RGG (C4) generators run in HBM (libslm
``slm_build_rmat`` / ``slm_build_rgg``), so the bench never moves the 1e9-entry edge list
over PCIe.  Their host twins -- the identical edge multisets, used as oracle and test inputs --
live outside the product, in ``workloads/`` (workloads/gen_host.c); the numpy-drawn SBM /
DC-SBM configs (C1, C2) exist only there and reach the device through
``Graph.from_edges`` / ``Context.build_graph``.
"""

from __future__ import annotations

import math

from . import _lib

RMAT_ABC = (0.57, 0.19, 0.19)


def rgg_radius(n, avg_deg=8.0):
    return math.sqrt(avg_deg / (math.pi * n))


def rmat_device(ctx: _lib.Context, scale, edge_factor, weight_mode=0, seed=0):
    """R-MAT (a, b, c) = RMAT_ABC, ids permuted, self-loops dropped, symmetrised, weights 1
    or U[1, 100] summed on duplicate merge; built as level 0 of ``ctx``."""
    ctx.build_rmat(scale, edge_factor, *RMAT_ABC, seed, weight_mode)


def rgg_device(ctx: _lib.Context, n, avg_deg=8.0, seed=0):
    """Random geometric graph, r = sqrt(avg_deg / (pi n)), unit weights; level 0 of ``ctx``."""
    ctx.build_rgg(n, rgg_radius(n, avg_deg), seed)


def sbm_device(ctx: _lib.Context, n, blocks, p_in, p_out, seed=0):
    """Planted-partition SBM drawn in HBM: one counter-hash Bernoulli draw per node pair
    (slm_build_pairs mode 0), blocks of n / blocks consecutive ids."""
    ctx.build_pairs(0, n, blocks, p_in, p_out, seed=seed)


def dcsbm_device(ctx: _lib.Context, params, seed=1):
    """Chung-Lu DC-SBM drawn in HBM (slm_build_pairs mode 1) over per-node parameters
    params = (comm, kin, kout, K, O) -- the O(n) parameters are host-side input, the O(n^2)
    pair draws run on the device."""
    ctx.build_pairs(1, len(params[0]), params=params, seed=seed)


def build_on_device(ctx: _lib.Context, spec: dict, edges=None):
    """Build a config described by ``spec`` (workloads.CONFIGS entry) as level 0 of ``ctx``:
    device-generated for R-MAT / RGG, from the host ``edges`` (n, src, dst, w) otherwise."""
    kind = spec["kind"]
    if kind == "rmat":
        rmat_device(ctx, spec["scale"], spec["edge_factor"], spec["weight_mode"], spec["seed"])
    elif kind == "rgg":
        rgg_device(ctx, spec["n"], spec["avg_deg"], spec["seed"])
    elif kind == "sbm_hash":
        sbm_device(ctx, spec["n"], spec["blocks"], spec["p_in"], spec["p_out"], spec["seed"])
    elif kind == "dcsbm_hash" and edges is not None and len(edges) == 5:
        dcsbm_device(ctx, edges, spec["seed"])   # edges = the pair-model parameters
    else:
        if edges is None:
            raise ValueError(f"config kind {kind!r} needs host edges")
        n, s, d, w = edges
        ctx.build_graph(n, s, d, w)
