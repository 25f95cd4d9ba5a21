mkdir -p gpurun_out
python -m pytest tests/test_gpu_fusion.py -x -q 2>&1 | tail -25 > gpurun_out/r2l_gputest.log
tail -3 gpurun_out/r2l_gputest.log
for fu in default combine2; do python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --fusion $fu > gpurun_out/r2l_c4_$fu.json 2>&1; python scripts/summ.py c4_$fu all < gpurun_out/r2l_c4_$fu.json; done
