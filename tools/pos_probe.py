"""Development probe: the first POSITIVE call of level 0 with the library's giant-part log."""
import os, sys, time
os.environ.setdefault("SLM_POS_LOG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1702_04645_b200 import _lib, generators as GN, RunConfig
ctx = _lib.Context(0)
GN.build_on_device(ctx, sys.argv[1] if len(sys.argv) > 1 else "c5_rmat24")
ctx.assign(want=False); ctx.components(want=False); ctx.sync()
t = time.perf_counter(); r = ctx.positive(RunConfig()._c()); ctx.sync()
print(f"positive0 {1e3*(time.perf_counter()-t):.1f} ms -> {r[:3]}", flush=True)
