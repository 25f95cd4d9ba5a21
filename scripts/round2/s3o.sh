# session 3: split-tf32 GEMMs with 8 split warps and shared-window loads: fp32 tests, c2 / c1 A/B
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "f32 or tf32 or fuzz" 2>&1 | tail -3 > gpurun_out/s3o_tests.log
for i in 1 2 3; do
python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/s3o_c2_$i.json 2>/dev/null
python bench.py --config c1 --no-cpu-baseline --no-e2e > gpurun_out/s3o_c1_$i.json 2>/dev/null
done
cat gpurun_out/s3o_tests.log
for f in gpurun_out/s3o_c*.json; do python scripts/summ.py $f < $f; done
