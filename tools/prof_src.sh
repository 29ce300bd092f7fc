#!/bin/bash
# Source-level capture of the sweep kernels: usage tools/prof_src.sh TAG [kernel-regex] [count]
TAG=${1:-dev}
KR=${2:-k_sweep}
CNT=${3:-9}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"$KR" -c $CNT -o gpurun_out/src_$TAG \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-partition > gpurun_out/ncu_src_$TAG.log 2>&1
echo SRC $?
