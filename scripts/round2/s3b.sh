# session 3: fused cached-mode dispatch (FUSE_CDISP) -- its tests, the cached tests, c5 A/B
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fusion.py tests/test_gpu_cache.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -8 > gpurun_out/s3b_tests.log
for i in 1 2 3; do
python bench.py --config c5 --fusion cdisp --no-cpu-baseline --no-e2e > gpurun_out/s3b_c5_cdisp_$i.json 2>/dev/null
python bench.py --config c5 --no-cpu-baseline --no-e2e --fusion default > gpurun_out/s3b_c5_nocdisp_$i.json 2>/dev/null
python bench.py --config c5 --alpha 1.0 --fusion cdisp --no-cpu-baseline --no-e2e > gpurun_out/s3b_c5s_cdisp_$i.json 2>/dev/null
python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/s3b_c3_$i.json 2>/dev/null
done
cat gpurun_out/s3b_tests.log
for f in gpurun_out/s3b_c*.json; do python scripts/summ.py $f all < $f; done
