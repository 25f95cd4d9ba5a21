# c3 / c5 bracketed on one box (caching evidence), c4 (k = 2) with and without O in token order
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-e2e"
$B --config c3 > gpurun_out/r2f_c3a.json 2>&1
$B --config c5 > gpurun_out/r2f_c5a.json 2>&1
$B --config c3 > gpurun_out/r2f_c3b.json 2>&1
$B --config c5 > gpurun_out/r2f_c5b.json 2>&1
$B --config c4 --steps 5 --warmup 3 > gpurun_out/r2f_c4_default.json 2>&1
$B --config c4 --steps 5 --warmup 3 --fusion legacy > gpurun_out/r2f_c4_legacy.json 2>&1
for f in gpurun_out/r2f_*.json; do python scripts/summ.py $(basename $f .json) all < $f; done
