mkdir -p gpurun_out
for v in 0 1 0 1; do MOE_DB1_IN_WGRAD=$v python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2n_db1w$v.json 2>&1; python scripts/summ.py db1w$v all < gpurun_out/r2n_db1w$v.json; done
MOE_DB1_IN_WGRAD=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fusion.py -x -q 2>&1 | tail -2
