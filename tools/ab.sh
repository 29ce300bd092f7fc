# A/B of the working library against build/libslm_base.so (development helper)
cd /root/repo
bash tools/quick.sh
for c in ${CFGS:-c5_rmat24}; do
for i in 1 2; do
 python tools/alloc_probe.py $c | grep ^run
 SLM_LIB_PATH=build/libslm_base.so python tools/alloc_probe.py $c | grep ^run
done
done
