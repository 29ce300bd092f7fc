python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t7_build.log 2>&1
for v in "SLM_CTA2=0" "SLM_CTA2=1" "SLM_CTA2_PRE=0"; do
  env $v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-partition --parity '' > gpurun_out/t7_bench_$v.json 2> gpurun_out/t7_bench_$v.err
done
