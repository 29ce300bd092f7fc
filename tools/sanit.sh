# NOTE (r02): compute-sanitizer is closed on the GPU pool ("runs under it have left GPUs
# needing a reset"); this recipe is kept for a box where it is available.
# compute-sanitizer evidence on small configs (profiles/r02_sanitizer_*.log): memcheck of a
# full level loop (every phase: build, ASSIGN, COMPONENTS, POSITIVE, MAXIMAL with the
# persistent commit walkers, AGGREGATE, score) and of the plan sweep / primitives;
# racecheck / synccheck of the same run (shared-memory hazards in the table kernels).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cat > /tmp/san_run.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, workloads as W, paper_1702_04645_b200 as P
for n, s, d, w in (W.rmat(11, 8, 1, 4), W.rgg(4096, 8.0, 3), W.generate("c1_sbm")):
    r = P.run(P.Graph.from_edges(n, s, d, w), P.RunConfig())
    print(n, r.stats.sweeps_per_level, r.final_score)
PY
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_run.py > gpurun_out/sanit_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanit_$tool.log
done
