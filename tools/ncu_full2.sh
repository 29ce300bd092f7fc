cd /root/repo
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_sweep_warp|k_sweep_half|k_sweep_cta" -c 5 -o gpurun_out/prof_sweep_r01h_b python bench.py --steps 1 --warmup 3 --no-cpu --no-partition > gpurun_out/ncu_full_r01h_b.log 2>&1; echo FULLB $?
grep -E "Profiling|ERROR" gpurun_out/ncu_full_r01h_b.log | head
