mkdir -p gpurun_out
MOE_BENCH_L2CLEAN=1 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench_l2clean.json 2>&1
python scripts/summ.py l2clean all < gpurun_out/r2d_bench_l2clean.json
KREGEX="combine_bwd|gate_fwd|gate_dw_tc" NAME=r2d_mem SKIP=3 COUNT=3 bash scripts/ncu_kernel.sh
ls -la gpurun_out
