mkdir -p gpurun_out
python -m pytest tests -m gpu -q -k "f32" 2>&1 | tail -25 > gpurun_out/r2h_gputest.log
tail -3 gpurun_out/r2h_gputest.log
for c in c1 c2; do python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/r2h_bench_$c.json 2>&1; python scripts/summ.py $c all < gpurun_out/r2h_bench_$c.json; done
