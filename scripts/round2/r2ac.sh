mkdir -p gpurun_out
python -m pytest tests -m gpu -q -k "f32" 2>&1 | tail -2
for i in 1 2; do
for c in c1 c2; do python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r2ac_${c}_$i.json 2>&1; python scripts/summ.py ${c} all < gpurun_out/r2ac_${c}_$i.json; done
python bench.py --config c2 --alpha 1.0 --no-cpu-baseline --no-e2e > gpurun_out/r2ac_c2s_$i.json 2>&1; python scripts/summ.py c2_static all < gpurun_out/r2ac_c2s_$i.json
done
