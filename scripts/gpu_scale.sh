mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scale.py -q -x -s > gpurun_out/t_scale.log 2>&1; echo scale=$?; tail -15 gpurun_out/t_scale.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sweep --no-c3 > gpurun_out/bench_c4.log 2>&1; echo bench=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_c4.log').read().strip().splitlines()[-1])
for k in ('value','ms_per_step','breakdown','e2e'):
    print(k, json.dumps(d.get(k)))
PY
