"""Development probe: context creation time (module preloading) and the first sweep's phases."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.cuda.init()
from paper_1702_04645_b200 import _lib
t = time.perf_counter(); ctx = _lib.Context(0); print(f"slm_create {1e3*(time.perf_counter()-t):.1f} ms", flush=True)
