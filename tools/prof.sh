#!/bin/bash
# GPU-box profiling recipe: bench line, launch list of the timed region (with DRAM bytes
# per launch), one full ncu capture of the sweep kernels.  usage: tools/prof.sh TAG [full]
TAG=${1:-dev}
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo BENCH $?
# timed region only (bench.py brackets it with cudaProfilerStart/Stop): 3 sweeps
ncu --profile-from-start off --clock-control none --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-partition > gpurun_out/ncu_launch_$TAG.log 2>&1
echo LAUNCH $?
if [ "$2" = "full" ]; then
  ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:"k_sweep|k_view" -c 16 -o gpurun_out/prof_sweep_$TAG \
      python bench.py --steps 1 --warmup 3 --no-cpu --no-partition > gpurun_out/ncu_full_$TAG.log 2>&1
  echo FULL $?
fi
