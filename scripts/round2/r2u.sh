mkdir -p gpurun_out
python bench.py --no-cpu-baseline --no-e2e --steps 300 --warmup 10 > gpurun_out/r2u_c3_sustained300.json 2>&1
python bench.py --no-cpu-baseline --no-e2e --graph > gpurun_out/r2u_c3_graph.json 2>&1
for i in 1 2; do
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2u_c3_$i.json 2>&1
python bench.py --no-cpu-baseline --no-e2e --config c5 --capacity static > gpurun_out/r2u_c5_static_$i.json 2>&1
done
for f in gpurun_out/r2u_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d['value'], d['ms_per_step'], d['step_ms']['median'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'), (d.get('graph') or {}))"; done
