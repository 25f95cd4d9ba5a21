# the bench's N = 4 path (c4 strong scaling, peer transport over IPC), ranks sharing one GPU
mkdir -p gpurun_out
MOE_BENCH_SHARE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/r2x_bench_n4.json 2> gpurun_out/r2x_bench_n4.err
echo rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/r2x_bench_n4.json').read().strip().splitlines()[-1])
print(d['value'], d['n_gpus'], d['ms_per_step'], d['config']['workload'], d['exchange'], d['device_flags'])"
tail -3 gpurun_out/r2x_bench_n4.err
