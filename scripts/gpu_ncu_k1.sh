mkdir -p gpurun_out
ONLY=INT8,INT4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:kv_append_kernel -c 2 -o gpurun_out/k1q python scripts/k1_once.py > gpurun_out/ncu_k1.log 2>&1; echo ncu=$?; tail -3 gpurun_out/ncu_k1.log
