mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/r2g_gputest.log
tail -3 gpurun_out/r2g_gputest.log
for c in c1 c2; do python bench.py --config $c --no-e2e > gpurun_out/r2g_bench_$c.json 2>&1; python scripts/summ.py $c all < gpurun_out/r2g_bench_$c.json; done
for c in c1 c2; do MOE_FORCE_SIMT=1 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/r2g_bench_${c}_simt.json 2>&1; python scripts/summ.py ${c}_simt all < gpurun_out/r2g_bench_${c}_simt.json; done
