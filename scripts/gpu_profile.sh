# ncu evidence for profiles/: launch list of the c4 bench's first eager steps
# (admission K1 + decode K2/merge at B=64) and one full capture of the
# dominant kernel (FP16 K2 at the c4 shape) and of the INT4 K2
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --profile > gpurun_out/prof_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'paged_decode_kernel<0' -c 1 -o gpurun_out/c4_fp16_full -f python bench.py --profile > gpurun_out/prof_full.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'paged_decode_kernel<3' -c 1 -o gpurun_out/c4_int4_full -f python bench.py --profile > gpurun_out/prof_full4.log 2>&1; echo ncu3=$?
ls -la gpurun_out | tail -5
