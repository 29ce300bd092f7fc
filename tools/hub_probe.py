"""Development probe: degree / distinct-community statistics of the rows of each degree bin
at the first MAXIMAL sweep's snapshot of a config (sizes the hub tables).  Not part of
the bench contract.   python tools/hub_probe.py [c5_rmat24]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1702_04645_b200 import _lib, generators as GN, RunConfig


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c5_rmat24"
    ctx = _lib.Context(0)
    GN.build_on_device(ctx, cfg)
    ctx.assign(want=False)
    ctx.components(want=False)
    ctx.positive(RunConfig()._c())
    _, comm, nc, _ = ctx.forest(want_a=False, want_cycle=False)
    lab = torch.from_numpy(comm.astype(np.int64)).cuda()
    n = comm.size
    p = np.empty(n + 1, np.int64)
    ctx.call("slm_get_union_rows", 0, n, _lib.ptr(p), None, None)
    deg = np.diff(p)
    edges = [0, 32, 256, 1024, 4096, 16383, 1 << 62]
    for b in range(6):
        rows = np.nonzero((deg > edges[b]) & (deg <= edges[b + 1]))[0]
        if rows.size == 0:
            continue
        samp = rows if rows.size <= 3000 else rows[np.linspace(0, rows.size - 1, 3000).astype(np.int64)]
        gs, ds = [], []
        for r in samp:
            p, nb, _ = ctx.union_rows(int(r), int(r) + 1)
            g = torch.unique(lab[torch.from_numpy(nb.astype(np.int64)).cuda()]).numel()
            gs.append(g)
            ds.append(nb.size)
        gs = np.array(gs); ds = np.array(ds)
        print(f"bin {b}: rows {rows.size} entries {deg[rows].sum()} | sample {samp.size}: "
              f"G/d {gs.sum()/ds.sum():.3f}  d max {ds.max()}  G max {gs.max()}  "
              f"d p50 {np.median(ds):.0f} G p50 {np.median(gs):.0f}", flush=True)
        if b == 5:
            o = np.argsort(-ds)[:12]
            print("   top d:", ds[o].tolist())
            print("   its G:", gs[o].tolist())
            print(f"   sum pow2(>d) slots {sum(1 << int(x).bit_length() for x in ds)}  "
                  f"sum pow2(>=2G) slots {sum(1 << int(2*x-1).bit_length() for x in gs)}")


if __name__ == "__main__":
    main()
