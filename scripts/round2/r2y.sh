mkdir -p gpurun_out
python -m pytest tests -m gpu -q -k "f32" 2>&1 | tail -3
for c in c1 c2; do python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r2y_$c.json 2>&1; python scripts/summ.py $c all < gpurun_out/r2y_$c.json; done
python bench.py --config c2 --alpha 1.0 --no-cpu-baseline --no-e2e > gpurun_out/r2y_c2_static.json 2>&1; python scripts/summ.py c2_static all < gpurun_out/r2y_c2_static.json
