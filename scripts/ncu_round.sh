#!/bin/bash
# ncu evidence for the current build (run on the GPU box via gpurun, 1 GPU).
# 1) launch list of every kernel of 2 bench steps (cold-cache, serialised: compare shares)
# 2) --set full captures of the expert GEMMs and of the memory-bound kernels.
set -x
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
BENCH="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BENCH > $OUT/ncu_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 6 -c 6 -o $OUT/prof_gemm -f $BENCH > $OUT/ncu_gemm.log 2>&1
# 9 memory-bound / small kernels per step (gate_fwd, route_hist, route_scan, dispatch,
# combine_bwd, bias_part_reduce, gate_dx, gate_dw, reduce_partials): skip the warm-up step
ncu --set full --clock-control none --import-source on -k regex:"dispatch|combine|colsum|gate_|zero_pad|route|reduce" -s 9 -c 9 -o $OUT/prof_mem -f $BENCH > $OUT/ncu_mem.log 2>&1
ls -la $OUT
