cd /root/repo
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r01h.log 2>&1; echo TESTS $(tail -1 gpurun_out/gpu_tests_r01h.log)
bash tools/prof.sh r01h
for c in c1_sbm c2_dcsbm c3_rmat22 c4_rgg24 c5_rmat24 c5_rmat24@0.5 c5_rmat24@2; do python tools/configs_run.py $c; done > gpurun_out/configs_r01h.jsonl 2> gpurun_out/configs_r01h.err; echo CFG $?
SLM_PRELOAD_MODULES=1 timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/late_sweep_r01h.csv python tools/sweep_kernels.py c5_rmat24 60 > gpurun_out/late_sweep_r01h.log 2>&1; echo LATE $?
python tools/launch_table.py gpurun_out/late_sweep_r01h.csv > gpurun_out/late_sweep_r01h.md
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE ok')"
cat gpurun_out/bench_r01h.json
