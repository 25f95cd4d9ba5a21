mkdir -p gpurun_out
for c in c2 c5; do python bench.py --config $c > gpurun_out/r2p_bench_$c.json 2> gpurun_out/r2p_bench_$c.err; python scripts/summ.py $c all < gpurun_out/r2p_bench_$c.json; tail -2 gpurun_out/r2p_bench_$c.err; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2p_bench_reference.json 2>&1; tail -c 600 gpurun_out/r2p_bench_reference.json
