python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t1_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -s > gpurun_out/t1_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/t1_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t1_smoke.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/t1_bench.json 2> gpurun_out/t1_bench.err
