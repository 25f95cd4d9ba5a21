# final evidence of the round-2 tree (after the backward tail): tests, smoke, bench lines,
# reference arm, launch list
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r2_final2_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final2_smoke.log 2>&1
python bench.py > gpurun_out/r2_final2_bench_c3.json 2> gpurun_out/r2_final2_bench_c3.err
python bench.py --config c2 > gpurun_out/r2_final2_bench_c2.json 2>/dev/null
python bench.py --config c2 --alpha 1.0 > gpurun_out/r2_final2_bench_c2_static.json 2>/dev/null
python bench.py --config c1 > gpurun_out/r2_final2_bench_c1.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
tail -2 gpurun_out/r2_final2_gputest.log; tail -3 gpurun_out/r2_final2_smoke.log
for c in c3 c2 c2_static c1; do python scripts/summ.py $c all < gpurun_out/r2_final2_bench_$c.json; done
