#!/bin/bash
# The paper's dynamic-capacity claim (fig:run-acc-gen) on B200: skewed routing
# (SPEC's clustered Gaussian), static alpha = 1.0 / 7.0 against the capacity policy
# (reading 14) after 50 warm-up steps, at c2 and c3.  One JSON line per run under $OUT.
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for cfg in c3 c2; do
  for mode in "static 1.0" "static 7.0" "dynamic 1.0"; do
    set -- $mode
    python bench.py --config $cfg --regime skewed --capacity $1 --alpha $2 --policy-warmup 50 \
      --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
      > $OUT/recompile_${cfg}_$1_$2.json 2> $OUT/recompile_${cfg}_$1_$2.err
  done
done
