# backward tail without PDL waits (MOE_TAIL) A/B, then the GPU tests
mkdir -p gpurun_out
for v in 1 0 1 0; do MOE_TAIL=$v python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2t_tail$v.json 2>&1; python scripts/summ.py tail$v all < gpurun_out/r2t_tail$v.json; python -c "
import json;d=json.loads(open('gpurun_out/r2t_tail$v.json').read().strip().splitlines()[-1]);print(d['value'], d['step_ms'], d['ms_per_step_profiled'])"; done
python -m pytest tests -m gpu -q 2>&1 | tail -3
