# session 3: weight-gradient k-tail trimming (skip the 16-deep MMAs of pad tokens): tests, A/B
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fusion.py -q -x -k "k_tail or half_tiles" 2>&1 | tail -4 > gpurun_out/s3k_tests.log
for i in 1 2 3; do
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s3k_c3_trim_$i.json 2>/dev/null
MOE_NO_KTRIM=1 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s3k_c3_notrim_$i.json 2>/dev/null
done
cat gpurun_out/s3k_tests.log
for f in gpurun_out/s3k_c3*.json; do python scripts/summ.py $f < $f; done
