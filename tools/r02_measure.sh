# Round-2 measurement recipe (one GPU box): tests, smoke, the bench's two arms, the ncu
# launch list of the timed region, one full ncu capture of the top sweep kernel, the
# end-to-end configs, sanitizers.  Outputs under gpurun_out/ (copied into profiles/).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${1:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 600 ncu --profile-from-start off --clock-control none --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-partition --parity '' > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"k_sweep_cta" --launch-skip 2 -c 1 -o gpurun_out/${T}_sweep_bin4_full \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-partition --parity '' > gpurun_out/${T}_ncu_full.log 2>&1
for c in c1_sbm c2_dcsbm c3_rmat22 c4_rgg24; do
  timeout 600 python tools/phase_compare.py $c >> gpurun_out/${T}_configs.jsonl 2>> gpurun_out/${T}_configs.err
done
for g in 1 0.5 2; do
  timeout 600 python tools/phase_compare.py c5_rmat24 $g >> gpurun_out/${T}_configs.jsonl 2>> gpurun_out/${T}_configs.err
done
# bash tools/sanit.sh   # (compute-sanitizer is closed on this GPU pool)
