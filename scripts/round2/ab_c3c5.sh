# alternating c3 / c5 (cached, static alpha 1) on one box: the caching gain
mkdir -p gpurun_out
for i in $(seq 1 ${N:-6}); do
  for c in c3 c5; do
    python bench.py --no-cpu-baseline --no-e2e --steps 30 --config $c --capacity static > gpurun_out/abc_${c}_${i}.json 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/abc_${c}_${i}.json').read().strip().splitlines()[-1])
print('$c', d['step_ms']['median'], d['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
