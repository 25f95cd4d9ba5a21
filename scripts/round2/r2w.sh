mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -3
N=6 bash scripts/round2/ab_c3c5.sh
