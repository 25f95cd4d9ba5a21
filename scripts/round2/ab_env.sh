# alternating A/B of an env switch: ENVVAR=<name> A=<value> B=<value> N=<pairs>
mkdir -p gpurun_out
for i in $(seq 1 ${N:-6}); do
  for v in $A $B; do
    env $ENVVAR=$v python bench.py --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/ab_${ENVVAR}_${v}_${i}.json 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/ab_${ENVVAR}_${v}_${i}.json').read().strip().splitlines()[-1])
print('$ENVVAR=$v', d['step_ms']['median'], d['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
