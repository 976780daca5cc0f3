for i in 1 2 3; do
  timeout 400 python bench.py --no-sweep --no-c3 --no-cpu-baseline > gpurun_out/b_hg.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/b_hg.log').read().strip().splitlines()[-1]);print(d['value'],d['breakdown']['admission_ms'], d['breakdown']['phase_change_ms_each'], d['breakdown']['step_ms_B8'], d['breakdown']['step_ms_B64'], d['e2e']['value'])" || tail -3 gpurun_out/b_hg.log
done
