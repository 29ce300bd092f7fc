python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p2_build.log 2>&1
export SLM_CTA2=0
timeout 900 ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --section InstructionStats --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_sweep_cta<512" -c 1 -o gpurun_out/p2_cta512 \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-partition --parity '' --scale 22 > gpurun_out/p2_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/p2_ncu.log
timeout 900 ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_sweep_warp" -c 1 -o gpurun_out/p2_warp \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-partition --parity '' --scale 22 >> gpurun_out/p2_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/p2_ncu.log
