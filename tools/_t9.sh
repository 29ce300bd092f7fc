python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t9_build.log 2>&1
for L in libslm_v1.so libslm.so; do
  SLM_LIB_PATH=$PWD/paper_1702_04645_b200/$L timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-partition --parity '' > gpurun_out/t9_bench_$L.json 2> gpurun_out/t9_bench_$L.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t9_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t9_tests.log
