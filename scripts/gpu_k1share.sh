for v in 0 1 2 3; do
KVSLAB_APPEND_PER_SM=$v timeout 400 python bench.py --no-sweep --no-c3 --no-cpu-baseline > gpurun_out/b_k1s.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/b_k1s.log').read().strip().splitlines()[-1]);print('$v', d['value'], d['breakdown']['admission_ms'], d['breakdown']['phase_change_ms_each'], {k:v['frac'] for k,v in d['k1_append'].items()})" || tail -3 gpurun_out/b_k1s.log
done
