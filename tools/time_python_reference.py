"""Times the real Python reference (synclouvain, installed offline into baseline/_ref) next
to the C oracle port and the B200 path on C1 / C2 (synclouvain.run at
threads=1 and threads=nproc), on the GPU box's host cores.  Checks that all three produce
the same hierarchy.  One JSON line per config.  (baseline/_ref is git-ignored and travels
with the repo snapshot; /root/reference is never read.)"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import numpy as np  # noqa: E402
import synclouvain as S  # noqa: E402
import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402

import paper_1702_04645_b200 as P  # noqa: E402

O.build()
nproc = os.cpu_count() or 1
O.set_threads(nproc)
for name in sys.argv[1:] or ["c1_sbm", "c2_dcsbm"]:
    n, s, d, w = W.generate(name)
    rec = {"config": name, "n": n, "edges": int(s.size), "cores": nproc}
    ref = None
    for t in (1, nproc):
        t0 = time.perf_counter()
        r = S.run(S.Graph.from_edges(n, s, d, w), S.RunConfig(threads=t))
        rec[f"python_reference_s_threads{t}"] = round(time.perf_counter() - t0, 3)
        ref = r
    t0 = time.perf_counter()
    o = O.run(n, s, d, w)
    rec["oracle_port_s"] = round(time.perf_counter() - t0, 3)
    P.run(P.Graph.from_edges(n, s, d, w), P.RunConfig())   # warm (module loads)
    t0 = time.perf_counter()
    g = P.run(P.Graph.from_edges(n, s, d, w), P.RunConfig())
    rec["b200_s"] = round(time.perf_counter() - t0, 3)
    same = lambda a, b: len(a) == len(b) and all(np.array_equal(x, y) for x, y in zip(a, b))
    rec["same_levels_reference_vs_b200"] = same(ref.hierarchy.levels, g.hierarchy.levels)
    rec["same_levels_reference_vs_oracle"] = same(ref.hierarchy.levels, o.levels)
    rec["modularity"] = g.final_score
    rec["sweeps_per_level"] = g.stats.sweeps_per_level
    print(json.dumps(rec), flush=True)
