# ncu evidence for profiles/: launch list of the c4 bench's first eager steps
# (admission K1 + decode K2/merge at B=64) and one full capture of each K2
# and K1 format at the c4 shape (the dominant kernel is FP16 K2)
set -x
mkdir -p gpurun_out
if [ -z "$SKIP_LIST" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --profile > gpurun_out/prof_launch.log 2>&1; echo ncu1=$?
fi
for k in ${KERNELS:-'paged_decode_kernel<.int.0,:c4_decode_fp16' 'paged_decode_kernel<.int.1,:c4_decode_fp8' 'paged_decode_kernel<.int.2,:c4_decode_int8' 'paged_decode_kernel<.int.3,:c4_decode_int4' 'kv_append_kernel<.int.0,:c4_k1_fp16' 'kv_append_kernel<.int.1,:c4_k1_fp8' 'kv_append_kernel<.int.2,:c4_k1_int8' 'kv_append_kernel<.int.3,:c4_k1_int4'}; do
  re=${k%%:*}; out=${k#*:}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$re" -c 1 -o gpurun_out/$out -f python bench.py --profile > gpurun_out/prof_$out.log 2>&1; echo $out=$?
done
ls -la gpurun_out/*.ncu-rep | tail -9
