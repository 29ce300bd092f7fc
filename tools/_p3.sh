python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p3_build.log 2>&1
timeout 900 ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --section InstructionStats --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_sweep_cta" -c 3 -o gpurun_out/p3_cta \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-partition --parity '' --scale 22 > gpurun_out/p3_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/p3_ncu.log
