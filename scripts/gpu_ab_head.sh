# A/B of the working tree's library against build_ab/H (HEAD), separate processes, alternated
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "$TESTS" > gpurun_out/ab_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/ab_tests.log
  grep -E "FAILED|Error|assert" gpurun_out/ab_tests.log | head -10
fi
for r in 1 2; do for v in new head; do
  if [ $v = head ]; then export KVSLAB_LIB_PATH=$PWD/build_ab/H/libkvslab.so; else unset KVSLAB_LIB_PATH; fi
  AB="{\"$v\":{}}" CASES=$CASES ROUNDS=3 timeout 300 python scripts/ab_decode.py 2>&1 | grep -v Warn
done; done | sort | tee gpurun_out/ab_head.log
