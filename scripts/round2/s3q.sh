# session 3 (reverted, the switch is gone): A-operand multicast across two CTA pairs
# (clusters of 4, MOE_TC_MC=1) with the pair-count grid (37 clusters): bitwise tests, c3 A/B
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_fusion.py -q -x -k "multicast" > gpurun_out/s3q_tests.log 2>&1
for i in 1 2 3; do for v in 0 1; do
MOE_TC_MC=$v timeout 120 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s3q_c3_mc${v}_$i.json 2>/dev/null
done; done
