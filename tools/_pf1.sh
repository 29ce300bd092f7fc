python -c "import __graft_entry__ as g; g.build()"
for a in "c3_rmat22 --scale 16" "c4_rgg24 --n 262144" "c5_rmat24 --scale 16 --gamma 0.5" "c5_rmat24 --scale 17 --gamma 2" "c2_dcsbm"; do
  timeout 900 python tools/parity_fullsize.py $a --lockstep -1 >> gpurun_out/pf1.jsonl 2>> gpurun_out/pf1.err
done
