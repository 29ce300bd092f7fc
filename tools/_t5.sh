python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t5_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_prims.py tests/test_gpu_parity.py -x -q > gpurun_out/t5_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t5_tests.log
timeout 300 python tools/prim_bench.py > gpurun_out/t5_prim.log 2>&1
timeout 300 python tools/phase_compare.py c5_rmat24 >> gpurun_out/t5_phase.jsonl 2>>gpurun_out/t5_phase.err
bash tools/_p1.sh
