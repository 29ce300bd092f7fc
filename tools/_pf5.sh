python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pf5_build.log 2>&1
timeout 3300 python tools/parity_fullsize.py c5_rmat24 --gamma 1 --lockstep -1 >> gpurun_out/pf5.jsonl 2>> gpurun_out/pf5.err
