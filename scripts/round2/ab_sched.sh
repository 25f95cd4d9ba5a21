mkdir -p gpurun_out
for i in 1 2 3; do for v in 0 1 2; do
MOE_TC_SCHED=$v python bench.py --no-cpu-baseline --no-e2e > gpurun_out/abs_${v}_${i}.json 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/abs_${v}_${i}.json').read().strip().splitlines()[-1])
k=d['kernels']; print('sched=$v', d['step_ms']['median'], d['ms_per_step'], {n:k[n]['avg_ms'] for n in ('ffn_gemm1','ffn_gemm2','wgrad_w2','dgrad_dA','wgrad_w1','dgrad_dX')})"
done; done
