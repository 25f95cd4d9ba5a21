# N > 1 path of the bench on one GPU (ranks share cuda:0 over a gloo group, peer transport
# over CUDA IPC): the c4 strong-scaling line at N = 2, and the reference arm at N = 2
mkdir -p gpurun_out
MOE_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2j_bench_n2.json 2> gpurun_out/r2j_bench_n2.err
tail -c 3000 gpurun_out/r2j_bench_n2.json
tail -5 gpurun_out/r2j_bench_n2.err
