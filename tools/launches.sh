#!/bin/bash
# per-kernel durations of bench.py's timed sweeps (3 sweeps): tools/launches.sh TAG [extra env]
TAG=${1:-dev}
timeout 600 ncu --profile-from-start off --clock-control none --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-partition > gpurun_out/ncu_launch_$TAG.log 2>&1
echo LAUNCH $?
python tools/summarize_launches.py gpurun_out/launches_$TAG.csv $TAG 3 2>&1 | tail -25
