#!/bin/bash
# ncu --set full of one kernel of the bench step (2nd step), with source correlation.
#   KREGEX=<kernel regex> NAME=<report name> [ENVS="A=1 B=2"] bash scripts/ncu_kernel.sh
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
env $ENVS ncu ${KBASE:+--kernel-name-base $KBASE} --set full --clock-control none --import-source on -k regex:"$KREGEX" -s ${SKIP:-1} -c ${COUNT:-1} \
  -o $OUT/$NAME -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > $OUT/$NAME.log 2>&1
