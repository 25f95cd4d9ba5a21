"""Expert-parallel path on one GPU: a 1-rank NCCL process group gives a real communicator,
so the whole EP machinery (count all-gather, host plan, grouped send/recv into the expert
regions, O / dO / dX return exchanges, fp32 all-reduce of dW_g) runs as a loopback and must
match both the oracle and the single-GPU path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle import moe_oracle as O
from parity_util import assert_routing_exact, assert_values, run_pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    from paper_2205_01848_b200.dist import nccl_comm_ptr
    yield nccl_comm_ptr()
    dist.destroy_process_group()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,k,renorm", [(8, 2, 1), (16, 1, 0)])
def test_ep_loopback_parity(comm, dtype, n, k, renorm):
    from paper_2205_01848_b200 import MoELayer
    T, d, f = 1000, 64, 128
    caps = O.capacities_from_factors([1.0] * n, T, k)
    ep = MoELayer(n, k, d, f, 0, T, dtype, renorm, world_size=1, rank=0, nccl_comm=comm,
                  device="cuda")
    layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, dtype, caps, renorm, layer=ep)
    assert st.routing.drops > 0
    assert_routing_exact(gpu, st, k, check_token_of_slot=False)
    assert_values(gpu, st, gr, ol, dtype)
    # the same numbers as the single-GPU path, bit for bit
    _, ref, _, _, _ = run_pair(n, k, d, f, T, dtype, caps, renorm)
    for key in ("y", "dx", "dw1", "db1", "dw2", "db2", "dw_gate"):
        assert np.array_equal(gpu[key], ref[key]), key


def test_ep_loopback_cached(comm):
    from paper_2205_01848_b200 import MoELayer
    from synth import perturb_cached
    n, k, T, d, f = 16, 2, 640, 64, 128
    caps = O.capacities_from_factors([1.25] * n, T, k)
    ep = MoELayer(n, k, d, f, 0, T, "bf16", 1, world_size=1, rank=0, nccl_comm=comm, device="cuda")
    layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, "bf16", caps, 1, layer=ep,
                                      cached=lambda fresh: perturb_cached(fresh, n, 0.03))
    assert_routing_exact(gpu, st, k, check_token_of_slot=False)
    assert_values(gpu, st, gr, ol, "bf16")
