"""Synchronised Louvain level loop (detector.py of the reference) over the B200 library.

``run(graph, RunConfig) -> RunResult`` keeps the reference's signature, stop rules and
statistics (detector.py:548-653).  The loop stays on the host, as in the reference; every
phase is one libslm call on device-resident state, and only per-level labels and scalars
cross the boundary.  ``RunConfig`` adds ``resolution`` (gamma), applied as m_w / gamma in
every gain; ``threads`` is accepted and ignored (the GPU grid replaces the
reference's row-chunk thread pool, detector.py:77-111).

Exact fast-forward: when a MAXIMAL sweep commits nothing, the forest is
unchanged, so the following POSITIVE call would return its own input (POSITIVE is
idempotent on its own output) with the same unresolved count; on integer-weight graphs it
is skipped and its statistics are replayed.  The device likewise reuses the sweep's plan while the forest is
unchanged and only redraws the coins.  Partitions, sweep counts and statistics are
identical to the reference's.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .forest import AssignmentForest, extract_components
from .graph import Graph, compose_labels

__all__ = ["Hierarchy", "RunConfig", "RunResult", "RunStats", "find_assignment",
           "maximal_correction", "positive_correction", "run"]


@dataclass(frozen=True)
class RunConfig:
    threads: int = 1
    seed: int = 0
    accept_prob: float = 0.5
    max_outer_iters: int = 100
    scc_cut_cap: int = 10_000
    debug_checks: bool = False
    record_scores: bool = False
    resolution: float = 1.0

    def __post_init__(self):   # detector.py:32-40
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if not (0.0 < self.accept_prob <= 1.0):
            raise ValueError("accept_prob must be in (0, 1]")
        if self.max_outer_iters < 1:
            raise ValueError("max_outer_iters must be >= 1")
        if self.scc_cut_cap < 2:
            raise ValueError("scc_cut_cap must be >= 2")
        if not (self.resolution > 0.0 and np.isfinite(self.resolution)):
            raise ValueError("resolution must be finite and > 0")

    def _c(self) -> _lib.SlmConfig:
        return _lib.SlmConfig(self.seed & ((1 << 64) - 1), float(self.accept_prob),
                              int(self.max_outer_iters), int(self.scc_cut_cap),
                              float(self.resolution))


@dataclass
class RunStats:
    levels: int = 0
    wall_seconds: float = 0.0
    sweeps_per_level: list = field(default_factory=list)
    accepted_moves: int = 0
    accepted_splits: int = 0
    unresolved_negative: int = 0
    phase_seconds: dict = field(default_factory=lambda: {
        k: 0.0 for k in ("assign", "components", "positive", "maximal", "aggregate")})
    score_trace: list = field(default_factory=list)
    trace_level_starts: list = field(default_factory=list)
    drift_checks: list = field(default_factory=list)
    warnings: list = field(default_factory=list)
    debug_failures: list = field(default_factory=list)
    skipped_positive_calls: int = 0     # exact fast-forward (not in the reference)
    plan_paths: list = field(default_factory=list)   # plan-sweep path per level (device)


@dataclass
class Hierarchy:
    levels: list
    flat: np.ndarray


@dataclass
class RunResult:
    hierarchy: Hierarchy
    final_score: float
    stats: RunStats


def _debug_validate(ctx: _lib.Context, phase: str, stats: RunStats, expect_clean_gains: bool):
    """detector.py:526-545 over state downloaded from the device."""
    a, comm, nc, oc = ctx.forest()
    ptr, nbr, _ = ctx.union()
    for i in np.flatnonzero(a != np.arange(a.size)).tolist():
        nb = nbr[ptr[i]:ptr[i + 1]]
        p = int(np.searchsorted(nb, a[i]))
        if p == nb.size or nb[p] != a[i]:
            stats.debug_failures.append(f"{phase}: node {i} points at non-neighbor {a[i]}")
    fresh = extract_components(a)
    if not (np.array_equal(fresh.comm, comm) and np.array_equal(fresh.on_cycle, oc)):
        stats.debug_failures.append(f"{phase}: stale component labeling")
    if expect_clean_gains:
        worst = float(ctx.local_gains().min()) if a.size else 0.0
        if worst < -1e-12:
            stats.debug_failures.append(f"{phase}: negative local gain {worst:.3e} left behind")


def run(graph: Graph, config: RunConfig | None = None) -> RunResult:
    """Detect communities and return the full level hierarchy (detector.py:548-653)."""
    if config is None:
        config = RunConfig()
    if graph.n == 0:
        raise ValueError("graph has no nodes")
    stats = RunStats()
    t_start = time.perf_counter()
    clock = {"t": t_start}

    def tick(phase):
        now = time.perf_counter()
        stats.phase_seconds[phase] += now - clock["t"]
        clock["t"] = now

    ctx = graph.context(level0=True)
    ctx.set_resolution(config.resolution)
    cfg = config._c()
    gamma = config.resolution
    if not (config.record_scores or config.debug_checks):
        # the whole loop below in one library call (slm_run): no host round trip per phase
        levels, sweeps, paths, capped, st, ph = ctx.run(cfg)
        stats.sweeps_per_level = sweeps
        stats.plan_paths = paths
        stats.accepted_moves, stats.accepted_splits, stats.unresolved_negative = (
            int(st[0]), int(st[1]), int(st[2]))
        stats.skipped_positive_calls = int(st[3])
        for t, c in enumerate(capped):
            if c:
                stats.warnings.append(f"level {t}: stopped after {config.max_outer_iters} sweeps")
        for k, v in zip(("assign", "components", "positive", "maximal", "aggregate"), ph):
            stats.phase_seconds[k] = float(v)
        flat = levels[0]
        for lv in levels[1:]:
            flat = compose_labels(flat, lv)
        final = ctx.score(flat, gamma, on_original=True)
        stats.levels = len(levels)
        stats.wall_seconds = time.perf_counter() - t_start
        return RunResult(hierarchy=Hierarchy(levels=levels, flat=flat), final_score=final,
                         stats=stats)
    trace = [] if config.record_scores else None
    want_g = trace is not None
    levels = []
    level = 0
    while True:
        info = ctx.info()
        n_level = info["n"]
        integral = info["integral"]
        stats.plan_paths.append(info["plan_path"])
        if trace is not None:
            stats.trace_level_starts.append(len(trace))
        clock["t"] = time.perf_counter()
        ctx.assign(want=False)
        tick("assign")
        comm, nc, _ = ctx.components(want=trace is not None)
        tick("components")
        running = ctx.score(comm, gamma, on_original=False) if trace is not None else 0.0
        _, splits, unresolved, gains = ctx.positive(cfg, want_gains=want_g)
        tick("positive")
        stats.accepted_splits += splits
        stats.unresolved_negative += unresolved
        last_unresolved = unresolved
        if trace is not None:
            for gv in gains:
                running += gv
                trace.append(running)
        if config.debug_checks:
            _debug_validate(ctx, f"positive@{level}", stats, unresolved == 0)
        sweeps = 0
        while True:
            if sweeps >= config.max_outer_iters:
                stats.warnings.append(f"level {level}: stopped after "
                                      f"{config.max_outer_iters} sweeps")
                break
            clock["t"] = time.perf_counter()
            improved, applied, gains = ctx.maximal(cfg, level, sweeps, want_gains=want_g)
            tick("maximal")
            sweeps += 1
            stats.accepted_moves += applied
            if trace is not None:
                for gv in gains:
                    running += gv
                    trace.append(running)
            if config.debug_checks:
                _debug_validate(ctx, f"maximal@{level}", stats, False)
            if not improved:
                break
            if applied == 0 and integral:
                # forest unchanged since the last POSITIVE, which is idempotent on its own
                # output: the call would change nothing and report the same unresolved count
                # (integer weights: local_gains' and the split's sums are exact, so their
                # signs agree; with real weights the call is made as in the reference)
                stats.unresolved_negative += last_unresolved
                stats.skipped_positive_calls += 1
                if config.debug_checks:
                    _debug_validate(ctx, f"positive@{level}", stats, last_unresolved == 0)
                continue
            _, splits, unresolved, gains = ctx.positive(cfg, want_gains=want_g)
            tick("positive")
            stats.accepted_splits += splits
            stats.unresolved_negative += unresolved
            last_unresolved = unresolved
            if trace is not None:
                for gv in gains:
                    running += gv
                    trace.append(running)
            if config.debug_checks:
                _debug_validate(ctx, f"positive@{level}", stats, unresolved == 0)
        stats.sweeps_per_level.append(sweeps)
        _, labels, nc, _ = ctx.forest(want_a=False, want_cycle=False)
        levels.append(labels)
        if trace is not None:
            exact = ctx.score(labels, gamma, on_original=False)
            stats.drift_checks.append((running, exact))
        if nc == n_level:
            break
        clock["t"] = time.perf_counter()
        ctx.aggregate()
        tick("aggregate")
        level += 1
    flat = levels[0]
    for lv in levels[1:]:
        flat = compose_labels(flat, lv)
    hierarchy = Hierarchy(levels=levels, flat=flat)
    final = ctx.score(flat, gamma, on_original=True)
    stats.levels = len(levels)
    if trace is not None:
        stats.score_trace = trace
    stats.wall_seconds = time.perf_counter() - t_start
    return RunResult(hierarchy=hierarchy, final_score=final, stats=stats)


# ------------------------------------------------------------------ phase mirrors

def find_assignment(graph: Graph, st=None, pool=None) -> np.ndarray:
    """detector.py:149-158 on the device."""
    return graph.context().assign()


def positive_correction(graph: Graph, st, forest: AssignmentForest, config: RunConfig, pool=None):
    """detector.py:338-362 -> (new_forest, splits, unresolved, gains)."""
    ctx = graph.context()
    ctx.set_resolution(config.resolution)
    ctx.set_assignment(forest.a)
    changed, splits, unresolved, gains = ctx.positive(config._c(), want_gains=True)
    if not changed:
        return forest, splits, unresolved, gains
    a, comm, nc, oc = ctx.forest()
    return AssignmentForest(a, comm, nc, oc), splits, unresolved, gains


def maximal_correction(graph: Graph, st, forest: AssignmentForest, config: RunConfig, level,
                       sweep, pool=None, stats=None):
    """detector.py:457-521 -> (new_forest, improved, applied, gains)."""
    ctx = graph.context()
    ctx.set_resolution(config.resolution)
    ctx.set_assignment(forest.a)
    improved, applied, gains = ctx.maximal(config._c(), level, sweep, want_gains=True)
    if not applied:
        return forest, improved, applied, gains
    a, comm, nc, oc = ctx.forest()
    return AssignmentForest(a, comm, nc, oc), improved, applied, gains
