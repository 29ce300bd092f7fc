python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p1_build.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_sweep_cta|k_sweep_warp|k_rs_onesweep|k_scan" -c 4 -o gpurun_out/p1_sweep \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-partition > gpurun_out/p1_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/p1_ncu.log
