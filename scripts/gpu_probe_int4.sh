mkdir -p gpurun_out
export KVSLAB_LIB_PATH=$PWD/build_ab/P/libkvslab.so
AB='{"full":{}, "compute_only":{"KVSLAB_DECODE_DEBUG":"4"}, "stream_only":{"KVSLAB_DECODE_DEBUG":"8"}}' \
CASES=INT4:64:4096,INT4:16:2048,FP8_E4M3:16:2048,INT8:16:2048,INT8:64:4096 ROUNDS=3 NOAPP=1 timeout 600 python scripts/ab_decode.py 2>&1 | grep -v Warn | tee gpurun_out/probe_int4.log
