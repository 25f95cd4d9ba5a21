mkdir -p gpurun_out
for i in 1 2; do for v in 1 0; do
MOE_TAIL=$v python bench.py --no-cpu-baseline --no-e2e --config c5 --capacity static > gpurun_out/r2v_c5_tail${v}_$i.json 2>&1
python scripts/summ.py c5_tail${v}_$i all < gpurun_out/r2v_c5_tail${v}_$i.json
done; done
