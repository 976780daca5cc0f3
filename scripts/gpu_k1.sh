mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/t_kernels.log 2>&1; echo kernels=$?; tail -2 gpurun_out/t_kernels.log
grep -E "^E .*differ|^FAILED" gpurun_out/t_kernels.log | head -5
for v in 0 1; do echo pipe=$v; KVSLAB_APPEND_PIPE=$v timeout 300 python scripts/bench_k1_k3.py 2>&1 | head -4; done
