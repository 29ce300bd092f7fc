"""Repeat-and-compare measurement (perf.py of the reference) for the device path.

``measure`` runs ``run()`` ``repeats`` times on one graph, raises ``DeterminismError`` when any
run's hierarchy differs bit for bit (perf.py:90-148), and writes ``runs.csv`` /
``phases.tsv`` in the reference's layout (perf.py:17-18, 140-147) with three extra columns
in runs.csv: the level-0 union entries, the plan-sweep rate in GTEPS and its fraction of the
HBM roofline (algorithmic bytes E*12 + n*32 + G*16 per sweep, over
MEASURED_PEAKS.json hbm_gbs or the 6,550 GB/s fallback).  ``threads`` is accepted and
ignored, as in RunConfig (the GPU grid replaces the thread pool).
"""

from __future__ import annotations

import csv
import json
import os
import time
from dataclasses import replace

import numpy as np

from .detector import RunConfig, run
from .graph import Graph

CSV_FIELDS = ("threads", "repeat", "wall_seconds", "score", "levels", "seed", "p",
              "union_entries", "plan_gteps", "plan_hbm_frac")
PHASES = ("assign", "components", "positive", "maximal", "aggregate")


class DeterminismError(RuntimeError):
    """Raised when repeated runs disagree on the partition (perf.py:21-22)."""


def hbm_peak_gbs() -> float:
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6550.0


def plan_rate(graph: Graph, config: RunConfig, sweeps: int = 5):
    """Device-timed plan sweeps on the first MAXIMAL sweep's level-0 snapshot ->
    (union entries, GTEPS, fraction of the HBM roofline)."""
    ctx = graph.context(level0=True)
    ctx.set_resolution(config.resolution)
    ctx.assign(want=False)
    ctx.components(want=False)
    ctx.positive(config._c())
    info = ctx.info()
    ctx.plan_async(127)
    ctx.sync()
    groups, _, _ = ctx.plan_groups()
    # the sweeps are queued back to back on the library stream; the host clock around the
    # synchronised batch is the device time up to one launch latency
    ctx.sync()
    t = time.perf_counter()
    for _ in range(sweeps):
        ctx.plan_async(127)
    ctx.sync()
    sec = (time.perf_counter() - t) / sweeps
    E, n = info["ue"], info["n"]
    gteps = E / sec / 1e9 if sec > 0 else 0.0
    B = E * 12 + n * 32 + groups * 16
    frac = B / sec / 1e9 / hbm_peak_gbs() if sec > 0 else 0.0
    return E, gteps, frac


def measure(graph: Graph, threads=(1,), repeats=2, config=None, csv_path=None,
            phase_path=None):
    """perf.py:90-148 on the device: repeated runs must agree bit for bit."""
    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    threads = sorted(set(int(t) for t in threads))
    base = config if config is not None else RunConfig()
    E, gteps, frac = plan_rate(graph, base)
    rows, ref = [], None
    phase_sums = {t: {k: 0.0 for k in PHASES} for t in threads}
    for t in threads:
        cfg = replace(base, threads=t)
        for rep in range(repeats):
            res = run(graph, cfg)
            if ref is None:
                ref = res.hierarchy
            elif not (np.array_equal(ref.flat, res.hierarchy.flat)
                      and len(ref.levels) == len(res.hierarchy.levels)
                      and all(np.array_equal(x, y) for x, y in zip(ref.levels, res.hierarchy.levels))):
                raise DeterminismError(f"partition changed at threads={t} repeat={rep}")
            for k in PHASES:
                phase_sums[t][k] += res.stats.phase_seconds[k]
            rows.append([t, rep, repr(res.stats.wall_seconds), repr(res.final_score),
                         res.stats.levels, cfg.seed, repr(cfg.accept_prob), E,
                         f"{gteps:.3f}", f"{frac:.4f}"])
    if csv_path is not None:
        with open(csv_path, "w", encoding="utf-8", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(CSV_FIELDS)
            w.writerows(rows)
    if phase_path is not None:
        with open(phase_path, "w", encoding="utf-8") as fh:
            fh.write("threads\tphase\tmean_seconds\n")
            for t in threads:
                for k in PHASES:
                    fh.write(f"{t}\t{k}\t{phase_sums[t][k] / repeats:.6f}\n")
    return rows


def amdahl(p_fraction: float, n_threads: int) -> float:
    """perf.py:53-60 (kept for the CLI's ``amdahl`` table)."""
    if not 0.0 <= p_fraction <= 1.0:
        raise ValueError("parallel fraction must lie in [0, 1]")
    if n_threads < 1:
        raise ValueError("thread count must be >= 1")
    return 1.0 / ((1.0 - p_fraction) + p_fraction / n_threads)
