"""Device generation of the BASELINE.json synthetic graphs straight into the level-0 build.

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


def build_on_device(ctx: _lib.Context, spec: dict, edges=None):
    """Build a config described by ``spec`` (workloads.CONFIGS entry) as level 0 of ``ctx``:
    device-generated for R-MAT / RGG, from the host ``edges`` (n, src, dst, w) otherwise."""
    kind = spec["kind"]
    if kind == "rmat":
        rmat_device(ctx, spec["scale"], spec["edge_factor"], spec["weight_mode"], spec["seed"])
    elif kind == "rgg":
        rgg_device(ctx, spec["n"], spec["avg_deg"], spec["seed"])
    else:
        if edges is None:
            raise ValueError(f"config kind {kind!r} needs host edges")
        n, s, d, w = edges
        ctx.build_graph(n, s, d, w)
