"""One device sort of 2^24 24-bit uint32 keys with int32 values (for an ncu launch list)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from paper_1702_04645_b200 import _lib  # noqa: E402

ctx = _lib.Context(0)
rng = np.random.default_rng(0)
n = 1 << 24
keys = rng.integers(0, 1 << 24, n, dtype=np.uint64).astype(np.uint32)
vals = np.arange(n, dtype=np.int32)
for _ in range(3):
    _, _, ms = ctx.debug_sort(keys, vals, 24)
print("sort ms", ms)
