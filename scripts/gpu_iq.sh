mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "decode" > gpurun_out/iq_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/iq_tests.log
grep -E "FAILED|Error|assert" gpurun_out/iq_tests.log | head -20
timeout 300 python scripts/acc_report.py 2>&1 | grep -v Warn | tee gpurun_out/iq_acc.log
# A/B against the HEAD build: separate processes (the library is bound at import), alternated
for r in 1 2; do for v in new head; do
  if [ $v = head ]; then export KVSLAB_LIB_PATH=$PWD/build_ab/H/libkvslab.so; else unset KVSLAB_LIB_PATH; fi
  AB="{\"$v\":{}}" CASES=${CASES:-INT4:64:4096,INT4:16:2048,INT4:8:8192,INT4:64:1300} ROUNDS=3 timeout 300 python scripts/ab_decode.py 2>&1 | grep -v Warn
done; done | sort | tee gpurun_out/iq_ab.log
