"""Development probe: per-sweep timing of the level loop (maximal / positive calls with the
library's phase split, SLM_PROFILE=1).  python tools/sweep_trace.py [config] [max_level]"""
import os
import sys
import time

os.environ.setdefault("SLM_PROFILE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_04645_b200 import _lib, generators as GN, RunConfig


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c5_rmat24"
    max_level = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    gamma = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    ctx = _lib.Context(0)
    GN.build_on_device(ctx, cfg_name)
    ctx.set_resolution(gamma)
    cfg = RunConfig()._c()
    level = 0
    while level <= max_level:
        n = ctx.info()["n"]
        ctx.assign(want=False)
        ctx.components(want=False)
        ctx.phase_times(reset=True)
        t = time.perf_counter()
        ctx.positive(cfg)
        print(f"L{level} n={n} positive0 {1e3*(time.perf_counter()-t):.1f} ms {ctx.phase_times(reset=True)}")
        sweeps = 0
        last = None
        tot = {"maximal": 0.0, "positive": 0.0}
        while sweeps < 100:
            t = time.perf_counter()
            imp, app, _ = ctx.maximal(cfg, level, sweeps)
            tm = 1e3 * (time.perf_counter() - t)
            pm = ctx.phase_times(reset=True)
            cand = ctx.last_commit_stats()
            sweeps += 1
            tot["maximal"] += tm
            tp = 0.0
            pp = {}
            if imp and app:
                t = time.perf_counter()
                ctx.positive(cfg)
                tp = 1e3 * (time.perf_counter() - t)
                pp = ctx.phase_times(reset=True)
                tot["positive"] += tp
            if sweeps <= 12 or sweeps % 10 == 0 or not imp:
                short = {k: round(v, 1) for k, v in pm.items() if v > 0.05}
                shortp = {k: round(v, 1) for k, v in pp.items() if v > 0.05}
                print(f"  s{sweeps-1:3d} applied {app:7d} cand/rounds {cand} max {tm:7.1f} ms {short} | pos {tp:6.1f} ms {shortp}")
            if not imp:
                break
        print(f"L{level} sweeps {sweeps} totals ms {tot}")
        ctx.aggregate()
        level += 1


if __name__ == "__main__":
    main()
