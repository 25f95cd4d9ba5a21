# session 3: fused cached-mode dispatch with TMA tile::scatter4 stores (code replaced by the register-staged copy, s3f) -- bitwise test, c5 A/B
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fusion.py -q -x -k "cached" 2>&1 | tail -4 > gpurun_out/s3e_tests.log
for i in 1 2; do
python bench.py --config c5 --fusion cdisp --no-cpu-baseline --no-e2e > gpurun_out/s3e_c5_cdisp_$i.json 2>/dev/null
python bench.py --config c5 --no-cpu-baseline --no-e2e --fusion default > gpurun_out/s3e_c5_nocdisp_$i.json 2>/dev/null
done
cat gpurun_out/s3e_tests.log
for f in gpurun_out/s3e_c*.json; do python scripts/summ.py $f all < $f; done
