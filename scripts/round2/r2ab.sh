mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -2
for i in 1 2 3; do for v in 1 0; do for c in c1 c2 c3; do
MOE_TAIL=$v python bench.py --config $c --alpha 1.0 --no-cpu-baseline --no-e2e > gpurun_out/r2ab_${c}_t${v}_$i.json 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/r2ab_${c}_t${v}_$i.json').read().strip().splitlines()[-1])
print('$c tail=$v', d['step_ms']['median'], d['ms_per_step'])"
done; done; done
