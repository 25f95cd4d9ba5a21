mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/r2i_gputest.log
tail -3 gpurun_out/r2i_gputest.log
for c in c1 c2; do python bench.py --config $c --graph > gpurun_out/r2i_bench_$c.json 2>&1; python scripts/summ.py $c all < gpurun_out/r2i_bench_$c.json; done
python bench.py > gpurun_out/r2i_bench_c3.json 2>&1; python scripts/summ.py c3 all < gpurun_out/r2i_bench_c3.json
