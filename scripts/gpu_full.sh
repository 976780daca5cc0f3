mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
grep -E "^FAILED|passed|failed|Error" gpurun_out/gpu_tests.log | head -20
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.log 2>&1; echo bench=$?
python - <<'PY'
import json
try:
    d=json.loads(open('gpurun_out/bench_full.log').read().strip().splitlines()[-1])
    for k in ('value','ms_per_step','decode_tok_s','breakdown','e2e','roofline','cpu_baseline','formats','gpu_launches','clocks'):
        print(k, json.dumps(d.get(k)))
    c3=d.get('c3',{}); print('c3', c3.get('value'), c3.get('breakdown'), json.dumps(c3.get('kernels')))
except Exception as e: print('parse', e); print(open('gpurun_out/bench_full.log').read()[-3000:])
PY
