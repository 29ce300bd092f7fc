python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t4_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t4_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t4_tests.log
timeout 300 python tools/prim_bench.py > gpurun_out/t4_prim.log 2>&1
SLM_PROFILE=1 timeout 300 python tools/phase_compare.py c5_rmat24 >> gpurun_out/t4_phase.jsonl 2>>gpurun_out/t4_phase.err
timeout 300 python tools/phase_compare.py c5_rmat24 >> gpurun_out/t4_phase.jsonl 2>>gpurun_out/t4_phase.err
SLM_LIB_PATH=$PWD/paper_1702_04645_b200/libslm_cub.so timeout 300 python tools/phase_compare.py c5_rmat24 >> gpurun_out/t4_phase.jsonl 2>>gpurun_out/t4_phase.err
