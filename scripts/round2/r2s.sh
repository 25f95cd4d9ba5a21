mkdir -p gpurun_out
for v in 0 2 4 6 0; do MOE_TC_DBG=$v python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2s_dbg$v.json 2>&1; python scripts/summ.py dbg$v < gpurun_out/r2s_dbg$v.json; done
