# A/B runs on the GPU box (round 2): GPU tests, then bench variants (per-kernel table)
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2}
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/${TAG}_gputest.log
for fu in ${FUSIONS:-default legacy}; do
python bench.py --no-cpu-baseline --no-e2e --fusion $fu > gpurun_out/${TAG}_bench_$fu.json 2>gpurun_out/${TAG}_bench_$fu.err
done
set +x
tail -3 gpurun_out/${TAG}_gputest.log
for f in gpurun_out/${TAG}_bench_*.json; do python scripts/summ.py $f all < $f; done
