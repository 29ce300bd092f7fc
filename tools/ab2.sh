# A/B across gammas (development helper)
cd /root/repo
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for g in 0.5 1; do
 python tools/alloc_probe.py c5_rmat24 $g | grep ^run
 SLM_LIB_PATH=build/libslm_base.so python tools/alloc_probe.py c5_rmat24 $g | grep ^run
done
python tools/alloc_probe.py c3_rmat22 | grep ^run
SLM_LIB_PATH=build/libslm_base.so python tools/alloc_probe.py c3_rmat22 | grep ^run
