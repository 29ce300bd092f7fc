"""Development run: full hierarchy of every BASELINE config on the GPU (device generator for
R-MAT / RGG, host generator otherwise), seconds to the final partition per config.
    python tools/configs_run.py [names...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_04645_b200 import _lib, detector, generators as GN, RunConfig
from paper_1702_04645_b200.graph import Graph


def run(name, gamma=1.0):
    ctx = _lib.Context(0)
    t0 = time.perf_counter()
    import workloads as W
    spec = W.CONFIGS[name]
    GN.build_on_device(ctx, spec, None if spec["kind"] in ("rmat", "rgg") else W.generate(name))
    tb = time.perf_counter() - t0
    info = ctx.info()
    g = Graph(info["n"], None, None, None)
    g._ctx = ctx
    ctx.level = 0
    t0 = time.perf_counter()
    r = detector.run(g, RunConfig(resolution=gamma))
    el = time.perf_counter() - t0
    return {"config": name, "gamma": gamma, "n": info["n"], "union_entries": info["ue"],
            "build_s": round(tb, 3), "run_s": round(el, 3), "levels": len(r.hierarchy.levels),
            "sweeps": r.stats.sweeps_per_level, "modularity": r.final_score,
            "phases": {k: round(v, 3) for k, v in r.stats.phase_seconds.items()}}


if __name__ == "__main__":
    names = sys.argv[1:] or ["c1_sbm", "c2_dcsbm", "c3_rmat22", "c4_rgg24", "c5_rmat24"]
    for nm in names:
        if "@" in nm:
            nm, gm = nm.split("@")
            print(json.dumps(run(nm, float(gm))), flush=True)
        else:
            print(json.dumps(run(nm)), flush=True)
