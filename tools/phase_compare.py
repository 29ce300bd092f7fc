"""A/B of the end-to-end level loop on a device-built config: seconds, phase seconds and the
library's own phase timers (SLM_PROFILE=1).  Usage: [SLM_LIB_PATH=...] python
tools/phase_compare.py c5_rmat24 [gamma]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from paper_1702_04645_b200 import RunConfig, _lib, detector, generators as GN  # noqa: E402
from paper_1702_04645_b200.graph import Graph  # noqa: E402

name = sys.argv[1]
gamma = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
spec = W.CONFIGS[name]
ctx = _lib.Context(0)
GN.build_on_device(ctx, spec, None if spec["kind"] in ("rmat", "rgg") else W.generate(name))
g = Graph(ctx.info()["n"], None, None, None)
g._ctx = ctx
ctx.phase_times(reset=True)
t = time.perf_counter()
r = detector.run(g, RunConfig(resolution=gamma))
el = time.perf_counter() - t
print(json.dumps({"lib": os.environ.get("SLM_LIB_PATH", "libslm.so"), "config": name,
                  "gamma": gamma, "seconds": round(el, 3), "sweeps": r.stats.sweeps_per_level, "plan_paths": r.stats.plan_paths,
                  "q": r.final_score,
                  "phase_s": {k: round(v, 3) for k, v in r.stats.phase_seconds.items()},
                  "lib_ms": ctx.phase_times()}))
