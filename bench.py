"""Bench: SLM local-move sweep (the plan sweep, _best_targets detector.py:367-418) on B200.

Contract (one JSON line from rank 0):
  * step    = one local-move plan sweep over the whole graph of the workload (default:
              BASELINE config 5, R-MAT scale 24, edge factor 32, integer weights U[1,100],
              ~1.02e9 directed union entries), on the snapshot the first MAXIMAL sweep of
              level 0 sees (after ASSIGN, COMPONENTS and POSITIVE).
  * value   = local-move GTEPS = union entries scanned per second, whole job (sum over ranks
              of entries / max over ranks of the device time of K sweeps; CUDA events on the
              library's own stream; inputs resident in HBM).  Inputs (12+ GB union) exceed
              the 126 MB L2, so no flush is needed between sweeps.
  * e2e     = the same metric through the reference-facing C ABI call with host buffers:
              slm_plan_sweep(labels from pinned host memory -> targets to host), H2D and D2H
              inside the timed region.
  * roofline: algorithmic bytes per sweep B = E*12 + n*32 + G*16 over the
              sweep's average device time, against MEASURED_PEAKS.json hbm_gbs.
  * cpu_baseline: the C oracle port of _best_targets on the host's cores over a bounded
              contiguous row sample of the same snapshot (also checked for equal targets);
              warm-up passes, then the mean over --steps passes.
  * --impl reference: the oracle port alone (the reference's CPU path), same metric and
              timing method, on a snapshot the oracle builds on the host from the workload's
              host twin (workloads/); the product package is never imported in that arm.
  * N > 1 (torchrun): replicas only: every rank runs the same sweep on
    its own GPU; rank 0 prints.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, device):
        self.device = device
        self.lines = []
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        self.t0 = self.t1 = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the sampler must be running before the timed region starts
            deadline = time.perf_counter() + 5.0
            while not self.lines and time.perf_counter() < deadline:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def start(self):
        self.t0 = time.perf_counter()

    def stop(self):
        self.t1 = time.perf_counter()
        time.sleep(0.12)   # the sample taken just after the last timed step

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append((time.perf_counter(), ln.strip()))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.t0 is not None and self.t1 is not None:
            # samples taken during the timed region (one sampling interval of slack at its
            # end); the first sample after its start when the region is shorter than that
            inside = [ln for t, ln in lines if self.t0 <= t <= self.t1 + 0.1]
            after = [ln for t, ln in lines if t >= self.t0][:1]
            lines = inside or after
        else:
            lines = [ln for _, ln in lines]
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def max_over_ranks(x: float, device="cpu") -> float:
    """Max of a per-rank scalar over the process group (no-op without one)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def _traffic():
    p = os.path.join(ROOT, "profiles", "plan_sweep_traffic.json")
    try:
        return json.load(open(p)).get("dram_bytes_per_sweep")
    except (OSError, ValueError):
        return None


def setup_snapshot(ctx, cfgname, over):
    """Build the workload in HBM and produce the first MAXIMAL sweep's snapshot."""
    import workloads as W
    from paper_1702_04645_b200 import RunConfig, generators as GN
    spec = {**W.CONFIGS[cfgname], **over}
    t0 = time.perf_counter()
    GN.build_on_device(ctx, spec, None if spec["kind"] in ("rmat", "rgg")
                       else W.generate(cfgname, **over))
    t1 = time.perf_counter()
    ctx.assign(want=False)
    ctx.components(want=False)
    ctx.positive(RunConfig()._c())
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


def snapshot_arrays(ctx):
    _, comm, nc, _ = ctx.forest(want_a=False, want_cycle=False)
    so, si, _ = ctx.aggregates(nc)
    return comm, so, si


def cpu_sample(ctx, info, target_entries, snap):
    """Download a contiguous row sample of the snapshot for the oracle port."""
    n = info["n"]
    # rows [0, R) with about target_entries union entries (the same rule as the reference
    # arm's oracle_snapshot: the graph's mean degree)
    avg = max(1.0, info["ue"] / max(1, n))
    R = int(min(n, max(1024, target_entries / avg)))
    uptr, unbr, uu = ctx.union_rows(0, R)
    comm, so, si = snap
    s_out, s_in, m = ctx.strengths()
    return dict(R=R, uptr=uptr, unbr=unbr, uu=uu, comm=comm, S_out=so, S_in=si, s_out=s_out,
                s_in=s_in, m=m, entries=int(uptr[-1]))


def time_oracle(sample, threads, warmup, steps):
    """The CPU plan sweep (_best_targets, oracle port) over the sample: ``warmup`` untimed
    passes, then the mean of ``steps`` timed passes -- the same method in the reference arm
    and in the ours-arm's cpu_baseline."""
    from oracle import oracle as O
    O.build()
    O.set_threads(threads)
    ts = []
    out = None
    for i in range(warmup + steps):
        t = time.perf_counter()
        out = O.plan_sample(sample["uptr"], sample["unbr"], sample["uu"], sample["s_out"],
                            sample["s_in"], sample["m"], sample["comm"], sample["S_out"],
                            sample["S_in"], 0, sample["R"])
        if i >= warmup:
            ts.append(time.perf_counter() - t)
    return sum(ts) / len(ts), out


def oracle_snapshot(cfgname, over, threads, target_entries):
    """Reference arm: the first MAXIMAL sweep's snapshot built on the host by the oracle
    (host twin of the workload -> Graph.from_edges -> ASSIGN -> COMPONENTS -> POSITIVE), and
    the bounded row sample the CPU plan sweep is timed on.  Nothing of the product is
    loaded."""
    import workloads as W
    from oracle import oracle as O
    O.build()
    O.set_threads(threads)
    t0 = time.perf_counter()
    n, s, d, w = W.generate(cfgname, **over)
    g = O.OGraph.from_edges(n, s, d, w)
    del s, d, w
    a = O.find_assignment(g)
    comm, nc, _ = O.extract_components(a)
    a, ch, *_ = O.positive_correction(g, a, comm, nc)
    if ch:
        comm, nc, _ = O.extract_components(a)
    so, si, _ = O.aggregates(g, comm, nc)
    uptr, unbr, uu = g.union()
    s_out, s_in, m = g.strengths()
    avg = max(1.0, uptr[-1] / max(1, n))
    R = int(min(n, max(1024, target_entries / avg)))
    sample = dict(R=R, uptr=uptr[:R + 1].copy(), unbr=unbr[:uptr[R]].copy(),
                  uu=uu[:uptr[R]].copy(), comm=comm, S_out=so, S_in=si, s_out=s_out,
                  s_in=s_in, m=m, entries=int(uptr[R]))
    return sample, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5_rmat24")
    ap.add_argument("--scale", type=int, default=None, help="override R-MAT scale (dev)")
    ap.add_argument("--cpu-entries", type=float, default=6e7,
                    help="union entries in the CPU-baseline row sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-partition", action="store_true",
                    help="skip the end-to-end seconds-to-final-partition runs")
    ap.add_argument("--parity", default="c3_rmat22",
                    help="comma list of configs checked against the oracle at full size, "
                         "full hierarchy in lockstep (tools/parity_fullsize.py); '' = none")
    ap.add_argument("--parity-timeout", type=float, default=900.0)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    ws, rank, local = _dist()
    import workloads as W
    over = {}
    if args.scale is not None:
        over["scale"] = args.scale
    spec = dict(W.CONFIGS[args.config])
    spec.update(over)
    workload = {"workload": args.config, **{k: v for k, v in spec.items()}}
    threads = os.cpu_count() or 1

    if args.impl == "reference":
        # the reference's CPU path (oracle port of _best_targets) on the host cores; the
        # snapshot is the oracle's own -- the product library is never imported here
        if ws > 1:
            import torch.distributed as dist
            dist.init_process_group(backend="gloo")
        if rank == 0:
            sample, prep_s = oracle_snapshot(args.config, over, threads, args.cpu_entries)
            t, _ = time_oracle(sample, threads, args.warmup, args.steps)
            val = sample["entries"] / t / 1e9
            line = {"impl": "reference", "metric": "local-move GTEPS", "value": val,
                    "unit": "GTEPS", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                    "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
                    "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                    "config": workload,
                    "cpu_baseline": {"value": val, "unit": "GTEPS", "cores": threads,
                                     "kind": "port",
                                     "sample": f"_best_targets over rows [0,{sample['R']}) "
                                               f"({sample['entries']} union entries) of the "
                                               f"{args.config} first-sweep snapshot (built by "
                                               f"the oracle on the host in {prep_s:.0f} s, "
                                               f"untimed)"},
                    "e2e": {"value": val, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                            "d2h_bytes_per_step": 0}}
            print(json.dumps(line), flush=True)
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return

    # full-size parity against the oracle (its own process, before this one reserves HBM)
    parity = parity_legs(args) if (rank == 0 and args.parity and not args.no_cpu) else None

    import torch
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group(backend="nccl")
    torch.cuda.set_device(local)
    from paper_1702_04645_b200 import _lib

    ctx = _lib.Context(local)
    build_s, setup_s = setup_snapshot(ctx, args.config, over)
    info = ctx.info()
    snap = snapshot_arrays(ctx)
    E, n = info["ue"], info["n"]
    # the first sweep of a level also builds the level's degree-ordered sweep view (once per
    # level, amortised over up to 100 sweeps): timed here, outside the timed steps
    ctx.sync()
    t0 = time.perf_counter()
    ctx.plan_async(127)
    ctx.sync()
    first_sweep_ms = (time.perf_counter() - t0) * 1e3

    groups, bin_rows, bin_entries = ctx.plan_groups()
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=local)
    # kernels per sweep (library launch sequence, slm_sweep.cu run_plan_u32): view labels in,
    # bin 0 (lane-per-row + packed), bin 1 (warp + half-warp rows), bins 2-4 (+ their
    # overflow pass), bin 5 (shared-table rows, global merge + select, fallback), targets out
    mid = int((bin_rows[2:5] > 0).sum())
    launches_per_sweep = (2 + 2 * int(bin_rows[0] > 0) + 2 * int(bin_rows[1] > 0) + mid
                          + int(mid > 0) + 4 * int(bin_rows[5] > 0))

    def timed(mask, iters):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(iters):
            ctx.plan_async(mask)
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b)

    for _ in range(args.warmup):
        ctx.plan_async(127)
    ctx.sync()
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    ctx.sync()
    # cudaProfilerStart/Stop bracket the timed sweeps so an
    # `ncu --profile-from-start off` launch list covers exactly the timed region
    torch.cuda.profiler.start()
    with Clocks(local) as clk:
        clk.start()
        ms = timed(127, args.steps)
        clk.stop()
    ctx.sync()
    torch.cuda.profiler.stop()
    torch.cuda.synchronize()
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    ms_max = max_over_ranks(ms, f"cuda:{local}")
    gpu_cstar = ctx.get_cstar()
    ms_step = ms_max / args.steps
    value = E * args.steps * ws / (ms_max / 1e3) / 1e9

    # per-bin device times (explanation only)
    per_bin = {}
    for mask, name in ((1, "bin0_lane_per_row_and_packed"), (2, "bin1_warp_hash512"),
                       (4, "bin2_cta128_hash2048"), (8, "bin3_cta256_hash2048"),
                       (16, "bin4_cta512_hash8192"), (32, "bin5_hub_smem_or_global"),
                       (64, "view_labels_in_targets_out")):
        if mask < 64 and bin_rows[mask.bit_length() - 1] == 0:
            continue
        per_bin[name] = round(timed(mask, max(3, args.steps // 4)) / max(3, args.steps // 4), 4)

    # e2e through the C ABI with pinned host buffers
    comm = snap[0]
    lab_pin = torch.from_numpy(comm).pin_memory().numpy()
    out_pin = torch.empty(n, dtype=torch.int64).pin_memory().numpy()
    from paper_1702_04645_b200._lib import ptr
    ke = args.steps
    ctx.call("slm_plan_sweep", ptr(lab_pin), ptr(out_pin))
    t0 = time.perf_counter()
    for _ in range(ke):
        ctx.call("slm_plan_sweep", ptr(lab_pin), ptr(out_pin))
    e2e_s = (time.perf_counter() - t0) / ke
    e2e_val = E * ws / e2e_s / 1e9

    # roofline of the sweep (SURVEY §8(d) algorithmic bytes)
    B = E * 12 + n * 32 + groups * 16
    peak, peak_kind = _peaks()
    achieved = B / (ms_step / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": _traffic(),
            "peak_kind": peak_kind, "algorithmic_bytes_per_sweep": int(B),
            "groups_G": int(groups), "G_over_E": round(groups / E, 4)}

    line = {"metric": "local-move GTEPS", "value": round(value, 3), "unit": "GTEPS",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {**workload, "n": n, "union_entries": E, "l2": "inputs > L2 (no flush)",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"},
            "roofline": roof,
            "e2e": {"value": round(e2e_val, 3), "unit": "GTEPS", "h2d_bytes_per_step": n * 8,
                    "d2h_bytes_per_step": n * 8, "ms_per_step": round(e2e_s * 1e3, 3)},
            "gpu_launches": launches_per_sweep * args.steps,
            "clocks": clk.summary(),
            "per_kernel_ms": per_bin,
            "bins": {"rows": bin_rows.tolist(), "entries": bin_entries.tolist()},
            "setup_s": {"build_csr_union": round(build_s, 3),
                        "assign_components_positive": round(setup_s, 3),
                        "first_sweep_ms": round(first_sweep_ms, 2),
                        # the level's degree-ordered sweep view (rows transposed into view
                        # order), built once per level by the first phase that sweeps the
                        # union -- here POSITIVE's local gains, inside the setup above
                        "sweep_view_build_ms": ctx.phase_times()["view_build_ms"]}}
    if rank == 0 and not args.no_cpu:
        sample = cpu_sample(ctx, info, args.cpu_entries, snap)
        t_cpu, cst = time_oracle(sample, threads, args.warmup, args.steps)
        ok = bool(np.array_equal(cst, gpu_cstar[:sample["R"]]))
        line["cpu_baseline"] = {
            "value": round(sample["entries"] / t_cpu / 1e9, 5), "unit": "GTEPS",
            "cores": threads, "kind": "port",
            "sample": f"_best_targets over rows [0,{sample['R']}) ({sample['entries']} union "
                      f"entries) of the same snapshot; targets equal to the GPU's: {ok}"}
    if not args.no_partition:
        line["partition"] = partition_runs(ctx, args, rank, threads)
    if parity is not None:
        line["parity"] = parity
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def parity_legs(args):
    """Full-size bit-exact parity (north_star: "partitions identical to the reference oracle
    on every integer-weighted config"): tools/parity_fullsize.py replays every phase of the
    device's level loop on the C oracle (host cores) from the same state, full hierarchy in
    lockstep, and reports the first mismatch if any."""
    out = {}
    for cfg in [c for c in args.parity.split(",") if c]:
        t0 = time.perf_counter()
        try:
            r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "parity_fullsize.py"),
                                cfg, "--lockstep", "-1"], capture_output=True, text=True,
                               timeout=args.parity_timeout)
            rec = json.loads(r.stdout.strip().splitlines()[-1])
            out[cfg] = {k: rec.get(k) for k in ("result", "phases_checked", "sweeps_per_level",
                                                "modularity", "modularity_oracle", "n",
                                                "union_entries", "oracle_threads")}
            out[cfg]["mode"] = "full hierarchy, every phase in lockstep"
        except subprocess.TimeoutExpired:
            out[cfg] = {"result": f"not finished within {args.parity_timeout:.0f} s"}
        except (ValueError, IndexError) as e:
            out[cfg] = {"result": f"harness error: {e}"}
        out[cfg]["seconds"] = round(time.perf_counter() - t0, 1)
    return out


def partition_runs(ctx, args, rank, threads):
    """BASELINE's second metric: end-to-end seconds to the final hierarchy.  (1) the workload
    config, graph already in HBM (device-generated), full level loop through the public
    run(); (2) C2 (DC-SBM, 10^5 nodes) from host edges through Graph.from_edges + run(),
    next to the C oracle's full hierarchy on the host cores (same partitions required)."""
    import workloads as W
    from paper_1702_04645_b200 import RunConfig, detector
    from paper_1702_04645_b200.graph import Graph
    out = {}
    info = ctx.info()
    g = Graph(info["n"], None, None, None)
    g._ctx = ctx
    ctx.level = 0
    torch_sync = __import__("torch").cuda.synchronize
    torch_sync()
    t0 = time.perf_counter()
    res = detector.run(g, RunConfig())
    el = time.perf_counter() - t0
    out[args.config] = {"seconds": round(el, 3), "levels": len(res.hierarchy.levels),
                        "sweeps_per_level": res.stats.sweeps_per_level,
                        "modularity": res.final_score,
                        "phase_seconds": {k: round(v, 3) for k, v in res.stats.phase_seconds.items()},
                        "input": "graph resident in HBM (device generator); timed: run()"}
    if rank == 0:
        n, s, d, w = W.generate("c2_dcsbm")
        t0 = time.perf_counter()
        g2 = Graph.from_edges(n, s, d, w)
        r2 = detector.run(g2, RunConfig())
        gpu_s = time.perf_counter() - t0
        c2 = {"seconds": round(gpu_s, 3), "levels": len(r2.hierarchy.levels),
              "modularity": r2.final_score,
              "input": "host edge list; timed: Graph.from_edges + run()"}
        if not args.no_cpu:
            from oracle import oracle as O
            O.build()
            O.set_threads(threads)
            t0 = time.perf_counter()
            ro = O.run(n, s, d, w)
            c2["cpu_port_seconds"] = round(time.perf_counter() - t0, 3)
            c2["cpu_cores"] = threads
            c2["same_partition"] = bool(
                len(ro.levels) == len(r2.hierarchy.levels)
                and all(np.array_equal(a, b) for a, b in zip(ro.levels, r2.hierarchy.levels)))
        out["c2_dcsbm"] = c2
    return out


if __name__ == "__main__":
    main()
