python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t6_build.log 2>&1
for v in 0 1; do
  SLM_CTA2=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-partition --parity '' > gpurun_out/t6_bench_cta2_$v.json 2> gpurun_out/t6_bench_cta2_$v.err
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t6_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t6_tests.log
