# memcheck of the sweep path on a mid-size R-MAT, and which sweep kernel fails under ncu replay
cd /root/repo
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python bench.py --steps 1 --warmup 3 --no-cpu --no-partition --scale 18 > gpurun_out/sanit.log 2>&1; echo SAN $?; grep -E "ERROR SUMMARY|Invalid|at 0x|by thread" gpurun_out/sanit.log | head -12
timeout 600 ncu --clock-control none --profile-from-start off -k regex:"k_sweep_warp|k_sweep_half|k_sweep_cta" -c 6 --metrics gpu__time_duration.sum python bench.py --steps 1 --warmup 3 --no-cpu --no-partition > gpurun_out/ncu_k.log 2>&1; echo NCU $?; grep -E "Profiling|ERROR" gpurun_out/ncu_k.log | head
