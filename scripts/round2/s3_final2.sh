# session-3 final evidence (re-run with the ncu reports kept outside gpurun_out/, which the
# first run overflowed): GPU tests with durations, smoke, bench lines, reference arm, ncu
# launch list + full-set summaries (written on the box, copied back)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=25 2>&1 | tail -32 > gpurun_out/s3_final_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_final_smoke.log 2>&1
python bench.py > gpurun_out/s3_final_bench_c3.json 2> gpurun_out/s3_final_bench_c3.err
python bench.py --config c5 --no-cpu-baseline > gpurun_out/s3_final_bench_c5.json 2>/dev/null
python bench.py --config c2 > gpurun_out/s3_final_bench_c2.json 2>/dev/null
python bench.py --config c1 > gpurun_out/s3_final_bench_c1.json 2>/dev/null
python bench.py --config c4 --no-cpu-baseline > gpurun_out/s3_final_bench_c4.json 2>/dev/null
python bench.py --impl reference > gpurun_out/s3_final_bench_reference.json 2>/dev/null
OUT=/tmp/ncu_s3 bash scripts/ncu_round.sh > /dev/null 2>&1
python scripts/ncu_summary.py s3_final /tmp/ncu_s3 > gpurun_out/s3_final_ncu_summary.log 2>&1
cp profiles/s3_final_ncu_full_summary.json profiles/s3_final_launches.txt profiles/ncu_traffic.json gpurun_out/ 2>/dev/null
ls -la /tmp/ncu_s3 >> gpurun_out/s3_final_ncu_summary.log
tail -3 gpurun_out/s3_final_gputest.log; tail -3 gpurun_out/s3_final_smoke.log
for c in c3 c5 c2 c1 c4; do python scripts/summ.py $c all < gpurun_out/s3_final_bench_$c.json; done
