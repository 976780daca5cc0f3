mkdir -p gpurun_out
CASE=INT4:64:4096 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'paged_decode_kernel<.int.3' -s 1 -c 1 -o gpurun_out/r02_iq_int4_b64 -f python scripts/one_decode.py > gpurun_out/ncu_iq.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_iq.log
