# session-3 closing check of the final tree (after the gate grid balance): GPU tests, smoke,
# c3 / c2 / c1 lines
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/s3_final4_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_final4_smoke.log 2>&1
python bench.py > gpurun_out/s3_final4_bench_c3.json 2>/dev/null
python bench.py --config c2 > gpurun_out/s3_final4_bench_c2.json 2>/dev/null
python bench.py --config c1 > gpurun_out/s3_final4_bench_c1.json 2>/dev/null
cat gpurun_out/s3_final4_gputest.log; tail -3 gpurun_out/s3_final4_smoke.log
for c in c3 c2 c1; do python scripts/summ.py $c < gpurun_out/s3_final4_bench_$c.json; done
