#!/bin/bash
# quick GPU check: gpu tests (log to gpurun_out/t.log) + bench per-bin line
timeout 600 python -m pytest tests -m gpu -x -q ${TESTK:+-k "$TESTK"} > gpurun_out/t.log 2>&1
echo "TESTS: $(tail -1 gpurun_out/t.log)"
timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu > gpurun_out/b.json 2> gpurun_out/b.err
echo "BENCH rc $?"
python3 - <<'PY'
import json
d = json.loads(open("gpurun_out/b.json").readline())
print(d["ms_per_step"], {k: round(v, 3) for k, v in d["per_kernel_ms"].items()})
PY
