mkdir -p gpurun_out
for w in c5 c1 c2; do
timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-sweep > gpurun_out/bench_$w.log 2>&1; echo $w=$?
python - $w <<'PY'
import json, sys
try:
    d=json.loads(open(f'gpurun_out/bench_{sys.argv[1]}.log').read().strip().splitlines()[-1])
    for k in ('value','ms_per_step','decode_tok_s','breakdown','per_gpu','roofline','e2e'):
        print(' ', k, json.dumps(d.get(k))[:400])
except Exception as e: print('parse', e); print(open(f'gpurun_out/bench_{sys.argv[1]}.log').read()[-2000:])
PY
done
