"""Development probe: build a config on the GPU, time each phase, print bin stats and a
full run's per-phase breakdown.  Not part of the bench contract.

    python tools/probe.py c5_rmat24 [--full] [--scale 20]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1702_04645_b200 import _lib, generators as GN, RunConfig


def ev_time(ctx, fn, iters=5):
    s = torch.cuda.ExternalStream(ctx.stream_ptr())
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    fn(); ctx.sync()
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(iters):
            fn()
        b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--max-sweeps", type=int, default=100)
    ap.add_argument("--no-maximal", action="store_true")
    a = ap.parse_args()
    over = {}
    if a.scale is not None:
        if "rmat" in a.config:
            over["scale"] = a.scale
        else:
            over["n"] = 1 << a.scale
    ctx = _lib.Context(0)
    t = time.perf_counter()
    GN.build_on_device(ctx, a.config, **over)
    ctx.phase_times(reset=True)
    info = ctx.info()
    print("build_s", round(time.perf_counter() - t, 3), json.dumps(info))
    t = time.perf_counter(); ctx.assign(want=False); print("assign_s", time.perf_counter() - t)
    t = time.perf_counter(); _, nc, _ = ctx.components(want=False); print("components_s", time.perf_counter() - t, "n_comms", nc)
    cfg = RunConfig()._c()
    t = time.perf_counter(); r = ctx.positive(cfg); print("positive_s", time.perf_counter() - t, r[:3])
    g, rows, ents = ctx.plan_groups()
    print("G", g, "G/E", g / info["ue"], "bin rows", rows.tolist(), "bin entries", ents.tolist())
    for mask, name in ((127, "sweep"), (1, "b0"), (2, "b1"), (4, "b2"), (8, "b3"), (16, "b4"), (32, "b5"), (64, "copy")):
        ms = ev_time(ctx, lambda: ctx.plan_async(mask))
        print(f"plan[{name}] ms {ms:.3f}  GTEPS(full E) {info['ue'] / ms / 1e6:.1f}")
    for mode in (0, 1, 2, 3, 4, 5):
        print("floor mode", mode, "ms", round(ctx.sweep_floor(mode), 3))
    if a.no_maximal:
        return
    t = time.perf_counter(); imp, app, _ = ctx.maximal(cfg, 0, 0); el = time.perf_counter() - t
    print("maximal0_s", el, "improved", imp, "applied", app, "cand/rounds", ctx.last_commit_stats())
    if a.full:
        from paper_1702_04645_b200.detector import run as _run
        from paper_1702_04645_b200.graph import Graph
        g = Graph(info["n"], None, None, None)
        g._ctx = ctx
        ctx.level = 0
        ctx.phase_times(reset=True)
        t = time.perf_counter()
        res = _run(g, RunConfig(max_outer_iters=a.max_sweeps))
        el = time.perf_counter() - t
        st = res.stats
        print("full_run_s", round(el, 3), "levels", st.levels, "sweeps", st.sweeps_per_level,
              "Q", res.final_score, "phase_s", {k: round(v, 3) for k, v in st.phase_seconds.items()},
              "moves", st.accepted_moves, "splits", st.accepted_splits, "skipped_pos", st.skipped_positive_calls)
        print("phase_ms", ctx.phase_times())


if __name__ == "__main__":
    main()
