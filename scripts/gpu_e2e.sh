timeout 400 python bench.py --no-sweep --no-c3 --no-cpu-baseline > gpurun_out/b_e2e.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/b_e2e.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step']*20, d['breakdown']); print(json.dumps(d['e2e']))" || tail -3 gpurun_out/b_e2e.log
