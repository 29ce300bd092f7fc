"""Development probe: how concentrated are the neighbour communities of a row?  For rows
[0, R) of the first MAXIMAL sweep's snapshot: fraction of union entries whose community is
the row's own, or one of the K largest communities, per degree bin.  Not part of the bench."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1702_04645_b200 import _lib, generators as GN, RunConfig


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c5_rmat24"
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
    ctx = _lib.Context(0)
    GN.build_on_device(ctx, cfg)
    ctx.assign(want=False)
    ctx.components(want=False)
    ctx.positive(RunConfig()._c())
    _, comm, nc, _ = ctx.forest(want_a=False, want_cycle=False)
    lab = torch.from_numpy(comm.astype(np.int64)).cuda()
    sizes = torch.bincount(lab, minlength=nc)
    top = torch.argsort(sizes, descending=True)[:8]
    print("n_comms", nc, "largest sizes", sizes[top].tolist())
    p, nb, _ = ctx.union_rows(0, R)
    p = torch.from_numpy(p.astype(np.int64)).cuda(); nb = torch.from_numpy(nb.astype(np.int64)).cuda()
    deg = p[1:] - p[:-1]
    row = torch.repeat_interleave(torch.arange(R, device="cuda"), deg)
    c = lab[nb]
    own = c == lab[row]
    edges = [0, 32, 256, 1024, 4096, 16383, 1 << 62]
    rb = torch.bucketize(deg, torch.tensor(edges[1:-1], device="cuda"), right=False)
    eb = rb[row]
    for b in range(6):
        m = eb == b
        ne = int(m.sum())
        if ne == 0:
            continue
        cc = c[m]
        res = [f"own {float(own[m].float().mean()):.3f}"]
        for k in (1, 2, 4, 8):
            res.append(f"top{k} {float(torch.isin(cc, top[:k]).float().mean()):.3f}")
        # share of the row's most frequent community (approx: top1 over whole graph excluded)
        print(f"bin {b}: entries {ne}", " ".join(res), flush=True)


if __name__ == "__main__":
    main()
