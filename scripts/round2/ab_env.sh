# alternating A/B of an env switch: ENVVAR=<name> A=<value> B=<value> N=<pairs> [CFG=<config>]
mkdir -p gpurun_out
for i in $(seq 1 ${N:-6}); do
  for v in $A $B; do
    out=gpurun_out/ab_${CFG:-c3}_${ENVVAR}_${v}_${i}.json
    env $ENVVAR=$v python bench.py --no-cpu-baseline --no-e2e --steps 30 ${CFG:+--config $CFG} > $out 2>&1
    python -c "
import json;d=json.loads(open('$out').read().strip().splitlines()[-1])
print('${CFG:-c3} $ENVVAR=$v', d['step_ms']['median'], d['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
