python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p4_build.log 2>&1
timeout 900 ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_sweep_cta" --launch-skip 2 -c 1 -o gpurun_out/p4_cta512 \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-partition --parity '' > gpurun_out/p4_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/p4_ncu.log
