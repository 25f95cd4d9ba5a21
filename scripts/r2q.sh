mkdir -p gpurun_out
for v in 0 1 0 1; do MOE_GDW_SPLIT=$v python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2q_split$v.json 2>&1; python scripts/summ.py split$v all < gpurun_out/r2q_split$v.json; python -c "
import json;d=json.loads(open('gpurun_out/r2q_split$v.json').read().strip().splitlines()[-1]);print(d['kernels']['gate_dw'], d['device_flags'], d['gpu_launches'])"; done
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
