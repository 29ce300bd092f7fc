python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t10_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t10_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t10_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t10_smoke.log 2>&1
timeout 900 python tools/time_python_reference.py c1_sbm c2_dcsbm > gpurun_out/t10_pyref.jsonl 2> gpurun_out/t10_pyref.err
