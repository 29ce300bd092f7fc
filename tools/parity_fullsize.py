"""Full-size parity of the B200 path against the C oracle (VERDICT r1 "next" item 1).

Runs the level loop of detector.py:548-653 on the device, phase by phase, and replays every
phase on the oracle from the SAME input state, diffing the outputs bit for bit:

  graph    level CSR / neighbour union / strengths / m_w (device build vs oracle
           Graph.from_edges at level 0, vs oracle aggregate() of the device labels above)
  ASSIGN   a                                    (detector.py:149-158)
  COMPS    comm, n_comms                        (forest.py:43-67)
  POSITIVE a, splits, unresolved, gains list    (detector.py:338-362)
  MAXIMAL  a, improved, applied, gains list     (detector.py:457-521)

``--lockstep K`` replays the first K sweeps of every level (K = -1: all of them, i.e. the
full hierarchy in lockstep, plus the flat partition and the final modularity); later
sweeps of a level run on the device alone, and the next level is again checked from the
device's labels (per-phase differential).  One JSON line per config on stdout.

Test / measurement infrastructure: it imports the oracle (only as the checker) and
workloads (host twins of the device generators).  Usage on the GPU box:
    python tools/parity_fullsize.py c3_rmat22 --lockstep -1
    python tools/parity_fullsize.py c5_rmat24 --gamma 0.5 --lockstep 2 --levels 2
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


class Mismatch(Exception):
    pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--gamma", type=float, default=1.0)
    ap.add_argument("--lockstep", type=int, default=-1,
                    help="sweeps per level replayed on the oracle (-1 = all)")
    ap.add_argument("--levels", type=int, default=-1,
                    help="levels checked (-1 = all); later levels run on the device alone")
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--graph-check", type=int, default=1)
    args = ap.parse_args()

    import workloads as W
    from oracle import oracle as O
    from paper_1702_04645_b200 import RunConfig, _lib, generators as GN
    O.build()
    O.set_threads(args.threads)
    over = {}
    if args.scale is not None:
        over["scale"] = args.scale
    if args.n is not None:
        over["n"] = args.n
    spec = {**W.CONFIGS[args.config], **over}
    cfg = RunConfig(resolution=args.gamma)
    cc = cfg._c()
    gamma = args.gamma
    log = {"config": args.config, **{k: v for k, v in over.items()}, "gamma": gamma,
           "lockstep": args.lockstep, "levels_checked": args.levels, "phases_checked": 0,
           "oracle_threads": args.threads}
    t_all = time.perf_counter()
    tick = {"gpu": 0.0, "oracle": 0.0, "compare": 0.0}

    def timed(key, fn, *a, **k):
        t = time.perf_counter()
        r = fn(*a, **k)
        tick[key] += time.perf_counter() - t
        return r

    def eq(name, x, y):
        t = time.perf_counter()
        ok = (np.array_equal(x, y) if isinstance(x, np.ndarray) or isinstance(y, np.ndarray)
              else x == y)
        tick["compare"] += time.perf_counter() - t
        log["phases_checked"] += 1
        if not ok:
            raise Mismatch(name)

    ctx = _lib.Context(0)
    t = time.perf_counter()
    edges = None
    if spec["kind"] in ("rmat", "rgg"):
        GN.build_on_device(ctx, spec)
    else:
        edges = W.generate(args.config, **over)
        GN.build_on_device(ctx, spec, edges)
    tick["gpu"] += time.perf_counter() - t
    ctx.set_resolution(gamma)
    if edges is None:
        edges = timed("oracle", W.generate, args.config, **over)
    n0, s0, d0, w0 = edges
    og = timed("oracle", O.OGraph.from_edges, n0, s0, d0, w0)
    del s0, d0, w0, edges
    og0 = og
    info = ctx.info()
    log.update(n=info["n"], union_entries=info["ue"])
    levels = []
    sweeps_pl = []
    try:
        level = 0
        while True:
            check = args.levels < 0 or level < args.levels
            n_level = ctx.info()["n"]
            if check and args.graph_check:
                # row chunks of ~2^26 entries (bounded host memory at 1e9 entries)
                step = max(1, int(n_level * (1 << 26) / max(1, og.ue)))
                for r0 in range(0, n_level, step):
                    r1 = min(n_level, r0 + step)
                    for which, nm, fg in ((0, "csr", ctx.csr_rows), (1, "union", ctx.union_rows)):
                        for part, x, y in zip(("ptr", "nbr", "w"), timed("gpu", fg, r0, r1),
                                              timed("oracle", og.rows, which, r0, r1)):
                            eq(f"L{level} {nm} {part} rows [{r0},{r1})", x, y)
                so_g, si_g, m_g = timed("gpu", ctx.strengths)
                so_o, si_o, m_o = timed("oracle", og.strengths)
                eq(f"L{level} s_out", so_g, so_o)
                eq(f"L{level} s_in", si_g, si_o)
                eq(f"L{level} m_w", m_g, m_o)
            m = og.m_w / gamma if check else None
            a_g = timed("gpu", ctx.assign, want=True)
            comm_g, nc_g, _ = timed("gpu", ctx.components, want=True)
            if check:
                a_o = timed("oracle", O.find_assignment, og, m)
                eq(f"L{level} assign", a_g, a_o)
                comm_o, nc_o, _ = timed("oracle", O.extract_components, a_o)
                eq(f"L{level} comm", comm_g, comm_o)
                eq(f"L{level} n_comms", nc_g, nc_o)

            def positive(tag, a_in, comm_in, nc_in, do_check):
                ch, sp, un, gains = timed("gpu", ctx.positive, cc, want_gains=do_check)
                if do_check:
                    a_g2 = timed("gpu", ctx.forest, want_comm=False, want_cycle=False)[0]
                    a_o2, ch_o, sp_o, un_o, gains_o, _ = timed(
                        "oracle", O.positive_correction, og, a_in, comm_in, nc_in,
                        cfg.scc_cut_cap, m)
                    eq(f"{tag} positive a", a_g2, a_o2)
                    eq(f"{tag} positive splits/unresolved", (sp, un), (sp_o, un_o))
                    eq(f"{tag} positive gains", np.asarray(gains, np.float64),
                       np.asarray(gains_o, np.float64))
                return un

            positive(f"L{level} first", a_g, comm_g, nc_g, check)
            last_un = None
            sweeps = 0
            while True:
                if sweeps >= cfg.max_outer_iters:
                    break
                lock = check and (args.lockstep < 0 or sweeps < args.lockstep)
                if lock:
                    a_in, comm_in, nc_in, _ = timed("gpu", ctx.forest, want_cycle=False)
                improved, applied, gains = timed("gpu", ctx.maximal, cc, level, sweeps,
                                                 want_gains=lock)
                if lock:
                    a_g2 = timed("gpu", ctx.forest, want_comm=False, want_cycle=False)[0]
                    a_o2, imp_o, app_o, gains_o, _ = timed(
                        "oracle", O.maximal_correction, og, a_in, comm_in, nc_in, cfg.seed,
                        cfg.accept_prob, level, sweeps, m)
                    eq(f"L{level} S{sweeps} maximal a", a_g2, a_o2)
                    eq(f"L{level} S{sweeps} maximal improved/applied", (improved, applied),
                       (imp_o, app_o))
                    eq(f"L{level} S{sweeps} maximal gains", np.asarray(gains, np.float64),
                       np.asarray(gains_o, np.float64))
                sweeps += 1
                if not improved:
                    break
                if applied == 0 and not lock:
                    continue   # exact skip (detector.run): forest unchanged since POSITIVE
                if lock:
                    a_in, comm_in, nc_in, _ = timed("gpu", ctx.forest, want_cycle=False)
                positive(f"L{level} S{sweeps - 1}", a_in if lock else None,
                         comm_in if lock else None, nc_in if lock else None, lock)
            sweeps_pl.append(sweeps)
            _, labels, nc, _ = ctx.forest(want_a=False, want_cycle=False)
            levels.append(labels)
            log.setdefault("levels_done", []).append(
                {"level": level, "n": n_level, "n_comms": nc, "sweeps": sweeps, "checked": check,
                 "elapsed_s": round(time.perf_counter() - t_all, 1)})
            print(json.dumps({"progress": log["levels_done"][-1]}), file=sys.stderr, flush=True)
            if nc == n_level:
                break
            timed("gpu", ctx.aggregate)
            if args.levels < 0 or level + 1 < args.levels:
                og = timed("oracle", O.aggregate, og, labels)
            level += 1
        flat = levels[0]
        for lv in levels[1:]:
            flat = lv[flat]
        q_g = ctx.score(flat, gamma, on_original=True)
        log["sweeps_per_level"] = sweeps_pl
        log["modularity"] = q_g
        if args.levels < 0:
            q_o = O.score(og0, flat, gamma)
            log["modularity_oracle"] = q_o
            eq("final modularity (1e-12 rel)", abs(q_g - q_o) <= 1e-12 * max(abs(q_o), 1e-300),
               True)
        log["result"] = "identical"
    except Mismatch as e:
        log["result"] = f"MISMATCH at {e}"
    log["seconds"] = {k: round(v, 1) for k, v in tick.items()}
    log["wall_s"] = round(time.perf_counter() - t_all, 1)
    print(json.dumps(log), flush=True)
    return 0 if log["result"] == "identical" else 1


if __name__ == "__main__":
    sys.exit(main())
