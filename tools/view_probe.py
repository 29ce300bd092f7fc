import os, sys, time
sys.path.insert(0, "/root/repo")
from paper_1702_04645_b200 import _lib, generators as GN, RunConfig
ctx = _lib.Context(0)
GN.build_on_device(ctx, "c5_rmat24")
cfg = RunConfig()._c()
for level in range(2):
    ctx.assign(want=False); ctx.components(want=False); ctx.positive(cfg)
    for k in range(2):
        t = time.perf_counter(); ctx.plan_async(127); ctx.sync(); print(f"L{level} plan {k}: {1e3*(time.perf_counter()-t):.1f} ms", flush=True)
    info = ctx.info(); print(info, flush=True)
    ctx.maximal(cfg, level, 0)
    ctx.aggregate()
