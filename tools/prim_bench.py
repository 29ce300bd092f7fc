"""Device primitives vs torch (CUB): stable pair sorts at the sizes the level loop uses."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1702_04645_b200 import _lib  # noqa: E402

ctx = _lib.Context(0)
rng = np.random.default_rng(0)


def tsort(keys, vals):
    kt = torch.from_numpy(keys.astype(np.int64)).cuda()
    vt = torch.from_numpy(vals).cuda()
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _, idx = torch.sort(kt, stable=True)
        vt[idx]
        b.record()
        b.synchronize()
    return a.elapsed_time(b)


for n, bits, kind in ((1 << 24, 24, 32), (1 << 24, 24, 64), (1 << 26, 48, 64), (1 << 20, 20, 32),
                      (1 << 16, 16, 32), (1 << 28, 48, 64)):
    if kind == 32:
        keys = rng.integers(0, 1 << bits, n, dtype=np.uint64).astype(np.uint32)
        vals = np.arange(n, dtype=np.int32)
    else:
        keys = rng.integers(0, 1 << bits, n, dtype=np.uint64)
        vals = rng.random(n)
    ctx.debug_sort(keys, vals, bits)
    _, _, ms = ctx.debug_sort(keys, vals, bits)
    print(f"n={n:>10} bits={bits} key{kind}: onesweep {ms:8.3f} ms   torch.sort+gather {tsort(keys, vals):8.3f} ms",
          flush=True)
