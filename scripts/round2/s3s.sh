# session 3 (reverted): split-tf32 GEMMs with 16-deep stages (64-byte swizzled K-major rows, twice the
# stages): every fp32 GPU test under a timeout, then c2 / c1 lines
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "f32 or tf32" > gpurun_out/s3s_tests.log 2>&1
echo "rc=$?" >> gpurun_out/s3s_tests.log
if grep -q " passed" gpurun_out/s3s_tests.log && ! grep -qE "failed|error" gpurun_out/s3s_tests.log; then
for i in 1 2 3; do
timeout 120 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/s3s_c2_$i.json 2>/dev/null
timeout 120 python bench.py --config c1 --no-cpu-baseline --no-e2e > gpurun_out/s3s_c1_$i.json 2>/dev/null
done
fi
tail -4 gpurun_out/s3s_tests.log
for f in gpurun_out/s3s_c*.json; do python scripts/summ.py $f < $f; done
