# A/B of the working library against build/libslm_base.so (development helper)
cd /root/repo
bash tools/quick.sh
python tools/pos_probe.py c5_rmat24 2>&1 | grep -E "section|slowest|positive0"
SLM_LIB_PATH=build/libslm_base.so python tools/pos_probe.py c5_rmat24 2>&1 | grep -E "section|slowest|positive0"
for i in 1 2; do
 python tools/alloc_probe.py ${CFG:-c5_rmat24} | grep ^run
 SLM_LIB_PATH=build/libslm_base.so python tools/alloc_probe.py ${CFG:-c5_rmat24} | grep ^run
done
