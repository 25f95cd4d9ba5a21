# session 3 (reverted, the switch is gone): 5 stages + two staging boxes per epilogue warp for FWD1 / DGRAD_A (MOE_TC2_STG2=1)
mkdir -p gpurun_out
MOE_TC2_STG2=1 python -m pytest tests/test_gpu_fusion.py tests/test_gpu_tc_gemm.py -q -x 2>&1 | tail -2 > gpurun_out/s3p_tests.log
for i in 1 2 3; do for v in 0 1; do
MOE_TC2_STG2=$v python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s3p_c3_stg2${v}_$i.json 2>/dev/null
done; done
cat gpurun_out/s3p_tests.log
for f in gpurun_out/s3p_c3*.json; do python scripts/summ.py $f < $f; done
