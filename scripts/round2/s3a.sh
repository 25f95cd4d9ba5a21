# session-3 re-entry check of the committed tree: GPU tests, smoke, c3 / c5 bench lines
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -6 > gpurun_out/s3a_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3a_smoke.log 2>&1
python bench.py > gpurun_out/s3a_bench_c3.json 2> gpurun_out/s3a_bench_c3.err
python bench.py --config c5 --no-cpu-baseline > gpurun_out/s3a_bench_c5.json 2>/dev/null
python bench.py --config c4 --no-cpu-baseline > gpurun_out/s3a_bench_c4.json 2>/dev/null
tail -2 gpurun_out/s3a_gputest.log; tail -3 gpurun_out/s3a_smoke.log
for c in c3 c5 c4; do python scripts/summ.py $c all < gpurun_out/s3a_bench_$c.json; done
