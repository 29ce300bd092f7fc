python -c "import __graft_entry__ as g; g.build()"
timeout 2700 python tools/parity_fullsize.py c4_rgg24 --lockstep -1 >> gpurun_out/pf2.jsonl 2>> gpurun_out/pf2.err
timeout 2700 python tools/parity_fullsize.py c3_rmat22 --lockstep -1 >> gpurun_out/pf2.jsonl 2>> gpurun_out/pf2.err
