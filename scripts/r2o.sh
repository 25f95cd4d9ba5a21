mkdir -p gpurun_out
for cfg in "0 0" "1 0" "1 1" "0 0" "1 0" "1 1"; do set -- $cfg
MOE_WBIAS_DIST=$1 MOE_DB1_IN_WGRAD=$2 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2o_d$1_w$2.json 2>&1; python scripts/summ.py d$1_w$2 all < gpurun_out/r2o_d$1_w$2.json; done
MOE_DB1_IN_WGRAD=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fusion.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fusion.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
