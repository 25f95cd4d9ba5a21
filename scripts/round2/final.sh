# final evidence of the round-2 tree: GPU tests, smoke, default bench line, reference arm
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r2_final_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final_smoke.log 2>&1
python bench.py > gpurun_out/r2_final_bench_c3.json 2> gpurun_out/r2_final_bench_c3.err
python bench.py --impl reference > gpurun_out/r2_final_bench_reference.json 2>&1
tail -2 gpurun_out/r2_final_gputest.log; tail -3 gpurun_out/r2_final_smoke.log
python scripts/summ.py c3 all < gpurun_out/r2_final_bench_c3.json
tail -c 400 gpurun_out/r2_final_bench_reference.json
