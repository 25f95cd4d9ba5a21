# session 3: caching at equal capacities on one box -- c3 vs c5 at static alpha = 1 (cached
# indices = the uncached run's routing), alternating, final tree
mkdir -p gpurun_out
for i in 1 2 3 4; do
python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/s3x_c3_$i.json 2>/dev/null
python bench.py --config c5 --alpha 1.0 --no-cpu-baseline --no-e2e > gpurun_out/s3x_c5a1_$i.json 2>/dev/null
done
for f in gpurun_out/s3x_*.json; do python scripts/summ.py $f all < $f | cut -c1-150; done
