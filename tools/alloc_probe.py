"""Development probe: host time in cudaMalloc/cudaFree during a full run (no profiling syncs)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_04645_b200 import _lib, detector, generators as GN, RunConfig
from paper_1702_04645_b200.graph import Graph
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5_rmat24"
ctx = _lib.Context(0)
GN.build_on_device(ctx, cfg)
print("build", ctx.phase_times(reset=True))
info = ctx.info(); g = Graph(info["n"], None, None, None); g._ctx = ctx; ctx.level = 0
gam = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
t = time.perf_counter(); r = detector.run(g, RunConfig(resolution=gam)); el = time.perf_counter() - t
pt = ctx.phase_times(reset=True)
print(f"run {el:.3f} s Q {r.final_score:.9f} alloc_ms {pt['alloc_ms']} calls {pt['alloc_calls']}", {k: round(v, 3) for k, v in r.stats.phase_seconds.items()})
if os.environ.get("SLM_PROFILE"):
    print("phase_ms", pt)
