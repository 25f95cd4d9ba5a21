# session 3 (reverted, the switch is gone): A-operand multicast, grid capped at the resident clusters of 4 (33 = 132 SMs); bitwise tests under a short
# timeout first, then c3 A/B
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_fusion.py -q -x -k "multicast" > gpurun_out/s3r_tests.log 2>&1
echo "rc=$?" >> gpurun_out/s3r_tests.log
if grep -q "passed" gpurun_out/s3r_tests.log && ! grep -q "failed" gpurun_out/s3r_tests.log; then
for i in 1 2; do for v in 0 1; do
MOE_TC_MC=$v timeout 120 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s3r_c3_mc${v}_$i.json 2>/dev/null
done; done
fi
tail -5 gpurun_out/s3r_tests.log
for f in gpurun_out/s3r_c3*.json; do python scripts/summ.py $f < $f; done
