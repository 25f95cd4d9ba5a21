# session 3 (reverted, the switch is gone): GEMM tile traversal direction A/B (MOE_TC_REV bit mask over FWD1, FWD2, WGRAD_W2,
# DGRAD_A, WGRAD_W1, DGRAD_X): a GEMM that starts on the rows its predecessor touched last
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fusion.py -q -x -k "bench_size" 2>&1 | tail -2 > gpurun_out/s3m_tests.log
MOE_TC_REV=0x3f python -m pytest tests/test_gpu_fusion.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2 >> gpurun_out/s3m_tests.log
for i in 1 2 3; do for m in 0 0x2a 0x15; do
MOE_TC_REV=$m python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s3m_c3_rev${m}_$i.json 2>/dev/null
done; done
cat gpurun_out/s3m_tests.log
for f in gpurun_out/s3m_c3*.json; do python scripts/summ.py $f < $f; done
