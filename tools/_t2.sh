python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t2_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t2_tests.log
timeout 300 python tools/prim_bench.py > gpurun_out/t2_prim.log 2>&1
for L in libslm_cub.so libslm.so; do
  SLM_PROFILE=1 SLM_LIB_PATH=$PWD/paper_1702_04645_b200/$L timeout 300 python tools/phase_compare.py c5_rmat24 >> gpurun_out/t2_phase.jsonl 2>>gpurun_out/t2_phase.err
  SLM_PROFILE=1 SLM_LIB_PATH=$PWD/paper_1702_04645_b200/$L timeout 300 python tools/phase_compare.py c3_rmat22 >> gpurun_out/t2_phase.jsonl 2>>gpurun_out/t2_phase.err
done
