"""Worker of tests/test_gpu_peer_ipc.py: one process per rank, each on its own GPU, the
peer-memory transport connected through CUDA IPC handles all-gathered over a gloo group;
each rank checks its shard of the outputs against the single-GPU layer bit for bit."""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    dist.init_process_group("gloo")
    R, r = dist.get_world_size(), dist.get_rank()
    dev = f"cuda:{r % torch.cuda.device_count()}"
    torch.cuda.set_device(dev)
    from oracle import moe_oracle as O
    from paper_2205_01848_b200 import MoELayer
    from paper_2205_01848_b200.dist import peer_connect
    from synth import make_dy, make_layer
    # IPC_SHAPE=ret: d = 128, top-1, raw weights -> return rows + fused dispatch backward
    ret = os.environ.get("IPC_SHAPE", "") == "ret"
    n, k, T, d, f, dtype = (8, 1, 256, 128, 256, "bf16") if ret else (8, 2, 256, 64, 128, "bf16")
    renorm = 0 if ret else 1
    Tg = R * T
    cpu = make_layer(n, d, f, d, Tg, dtype)
    g = {kk: v.cuda() for kk, v in cpu.items()}
    dy = make_dy(Tg, d, dtype).cuda()
    caps = O.capacities_from_factors([1.0] * n, Tg, k)
    L = MoELayer(n, k, d, f, 0, T, dtype, renorm, world_size=R, rank=r, device=dev,
                 transport="peer")
    peer_connect(L)
    L.set_capacities(caps)
    for _ in range(2):
        y = L.forward(g["x"][r * T:(r + 1) * T], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
        gr = L.backward(dy[r * T:(r + 1) * T].contiguous())
    torch.cuda.synchronize()
    ref = MoELayer(n, k, d, f, 0, Tg, dtype, renorm, device=dev)
    ref.set_capacities(caps)
    y_ref = ref.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    gr_ref = ref.backward(dy)
    torch.cuda.synchronize()
    ok = torch.equal(y, y_ref[r * T:(r + 1) * T]) and torch.equal(gr["dx"], gr_ref["dx"][r * T:(r + 1) * T])
    nl = n // R
    for key in ("dw1", "db1", "dw2", "db2"):
        ok = ok and torch.equal(gr[key][r * nl:(r + 1) * nl], gr_ref[key][r * nl:(r + 1) * nl])
    dist.barrier()
    L.close()
    dist.destroy_process_group()
    print(f"rank {r}: {'OK' if ok else 'MISMATCH'}", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
