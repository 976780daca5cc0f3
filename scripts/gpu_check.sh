# quick GPU iteration: parity tests + bench (no CPU leg)
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
grep -E "^FAILED|passed|failed|Error" gpurun_out/gpu_tests.log | head -20
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -3 gpurun_out/bench.log
