cd /root/repo
bash tools/quick.sh
for i in 1 2; do
 python tools/alloc_probe.py c5_rmat24 | grep ^run
 SLM_LIB_PATH=build/libslm_base.so python tools/alloc_probe.py c5_rmat24 | grep ^run
done
python tools/alloc_probe.py c3_rmat22 | grep ^run
SLM_LIB_PATH=build/libslm_base.so python tools/alloc_probe.py c3_rmat22 | grep ^run
