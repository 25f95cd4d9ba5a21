# half tiles: correctness first, then alternating A/B on c5 (dynamic), c2 (dynamic), c3
set -x
python -m pytest tests/test_gpu_fusion.py -x -q -k half_tiles 2>&1 | tail -5
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in c5 c2 c3; do CFG=$c ENVVAR=MOE_HALF_TILES A=1 B=0 N=4 bash scripts/round2/ab_env.sh; done
