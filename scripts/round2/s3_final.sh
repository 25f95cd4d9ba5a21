# session-3 final evidence of the round-2 tree: GPU tests, smoke, bench lines (c3 default args,
# c5, c2, c1, c4), reference arm, ncu launch list + full-set captures (scripts/ncu_round.sh)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/s3_final_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_final_smoke.log 2>&1
python bench.py > gpurun_out/s3_final_bench_c3.json 2> gpurun_out/s3_final_bench_c3.err
python bench.py --config c5 --no-cpu-baseline > gpurun_out/s3_final_bench_c5.json 2>/dev/null
python bench.py --config c2 > gpurun_out/s3_final_bench_c2.json 2>/dev/null
python bench.py --config c1 > gpurun_out/s3_final_bench_c1.json 2>/dev/null
python bench.py --config c4 --no-cpu-baseline > gpurun_out/s3_final_bench_c4.json 2>/dev/null
python bench.py --impl reference > gpurun_out/s3_final_bench_reference.json 2>/dev/null
bash scripts/ncu_round.sh > /dev/null 2>&1
tail -2 gpurun_out/s3_final_gputest.log; tail -3 gpurun_out/s3_final_smoke.log
for c in c3 c5 c2 c1 c4; do python scripts/summ.py $c all < gpurun_out/s3_final_bench_$c.json; done
head -c 600 gpurun_out/s3_final_bench_reference.json
