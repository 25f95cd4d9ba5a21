mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/r2k_gputest.log
tail -3 gpurun_out/r2k_gputest.log
python bench.py --no-cpu-baseline --no-e2e --ep > gpurun_out/r2k_bench_ep1.json 2>&1; python scripts/summ.py ep1 all < gpurun_out/r2k_bench_ep1.json
