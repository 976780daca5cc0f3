set -x
#timeout 600 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
grep -E "^FAILED|passed|failed" gpurun_out/gpu_tests.log
#timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'paged_decode|kv_append' -c 256 --csv --log-file gpurun_out/launches.csv python bench.py --profile > gpurun_out/prof_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_decode -c 2 -o gpurun_out/decode_full python bench.py --profile > gpurun_out/prof_full.log 2>&1; echo ncu2=$?
ls -la gpurun_out
