timeout 400 python bench.py --no-sweep --no-c3 --no-cpu-baseline > gpurun_out/b_t.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/b_t.log').read().strip().splitlines()[-1]);print(d['value'], d['breakdown']['step_ms_B8'], d['breakdown']['step_ms_B64']); print(json.dumps(d['sm_share']))" || tail -3 gpurun_out/b_t.log
