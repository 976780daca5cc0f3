# quick GPU iteration (scratch): K1 parity + K1/K3 probe + bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/t_kernels.log 2>&1; echo kernels=$?; tail -2 gpurun_out/t_kernels.log
timeout 300 python scripts/bench_k1_k3.py 2>&1 | head -4
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sweep ${BENCH_ARGS} > gpurun_out/bench_c4.log 2>&1; echo bench=$?; python - <<'PY'
import json
try:
    d=json.loads(open('gpurun_out/bench_c4.log').read().strip().splitlines()[-1])
    for k in ('value','ms_per_step','decode_tok_s','frac_of_peak','breakdown','e2e','kernels','c4'):
        print(k, json.dumps(d.get(k)))
    c3=d.get('c3',{}); print('c3', c3.get('value'), c3.get('breakdown'), json.dumps(c3.get('e2e')))
except Exception as e: print('parse', e); print(open('gpurun_out/bench_c4.log').read()[-3000:])
PY
