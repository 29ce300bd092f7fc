"""Development probe: run level 0 of a config up to a late sweep, then bracket one maximal +
positive call with cudaProfilerStart/Stop (for an `ncu --profile-from-start off` launch list
of one whole late sweep).  python tools/sweep_kernels.py [config] [sweep]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1702_04645_b200 import _lib, generators as GN, RunConfig
cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c5_rmat24"
target = int(sys.argv[2]) if len(sys.argv) > 2 else 60
ctx = _lib.Context(0)
import workloads as W
spec = W.CONFIGS[cfg_name]
GN.build_on_device(ctx, spec, None if spec["kind"] in ("rmat", "rgg") else W.generate(cfg_name))
cfg = RunConfig()._c()
ctx.assign(want=False); ctx.components(want=False); ctx.positive(cfg)
for sw in range(target + 1):
    last = sw == target
    if last:
        ctx.sync(); torch.cuda.profiler.start()
    imp, app, _ = ctx.maximal(cfg, 0, sw)
    if imp and app:
        ctx.positive(cfg)
    if last:
        ctx.sync(); torch.cuda.profiler.stop()
print("done", sw, app)
