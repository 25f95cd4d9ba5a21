"""Expert-parallel host logic on CPU with world_size-2 gloo process groups.

Each rank routes its own slice of a shared seeded batch (oracle top-k), the per-rank counts
are all-gathered over gloo, and the library's moe_ep_plan must (a) be identical on every rank,
(b) give message sizes that match pairwise (what r sends to owner(e) is what the owner
expects from r), and (c) reproduce the oracle's GLOBAL routing (reading 12): the kept pairs
and global slots of the concatenated batch.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import moe_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _plan(lib, R, rank, n, cnt_all, cap):
    arr = lambda m, t=C.c_int32: (t * m)()  # noqa: E731
    cin = (C.c_int32 * (R * n))(*cnt_all.reshape(-1).tolist())
    cc = (C.c_int32 * n)(*cap)
    pre, kl, so, kloc, dr = arr(R * n), arr(R * n), arr(n), arr(n // R), (C.c_int64 * 1)()
    assert lib.moe_ep_plan(R, rank, n, cin, cc, pre, kl, so, kloc, dr) == 0
    return (np.array(pre).reshape(R, n), np.array(kl).reshape(R, n), np.array(so),
            np.array(kloc), int(dr[0]))


def _worker(rank, R, port, n, k, T, cap, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=R)
    from paper_2205_01848_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(5)
    logits = rng.standard_normal((R * T, n))          # the shared global batch
    idx = O.topk_sorted(logits[rank * T:(rank + 1) * T], k)
    local = O.route(idx, [10**9] * n, n).counts.astype(np.int32)
    g = [torch.zeros(n, dtype=torch.int32) for _ in range(R)]
    dist.all_gather(g, torch.from_numpy(local))
    cnt_all = torch.stack(g).numpy()
    pre, kl, so, kloc, drops = _plan(lib, R, rank, n, cnt_all, cap)
    # the plan is identical on all ranks
    out = [None] * R
    dist.all_gather_object(out, (pre.tolist(), kl.tolist(), drops))
    # oracle: this rank's slice routed with the prior counts of lower ranks == global routing
    glob = O.route(O.topk_sorted(logits, k), cap, n)
    part = O.route(idx, cap, n, token_offset=rank * T, prior_counts=pre[rank])
    ok_slots = np.array_equal(part.slot_of, glob.slot_of[rank * T:(rank + 1) * T])
    ok_kl = np.array_equal(kl[rank], part.kept)
    q.put((rank, out, ok_slots, ok_kl, kloc.tolist(), so.tolist(), drops, glob.drops,
           glob.kept.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("R,n,k", [(2, 8, 2), (2, 6, 1)])
def test_ep_plan_gloo_world2(R, n, k):
    from paper_2205_01848_b200 import _lib, build
    if not os.path.exists(_lib.LIB_PATH):
        build.build()
    T = 300
    cap = O.capacities_from_factors([1.0] * n, R * T, k)
    cap[1] = 5                                              # force drops on one expert
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, R, port, n, k, T, cap, q)) for r in range(R)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(R)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    plans = [r[1] for r in res]
    for r in res:
        assert r[1] == plans[0]                             # identical on every rank
        assert r[2] and r[3]                                # global slots / kept pairs
        assert r[6] == r[7]                                 # drops == oracle global drops
    # kept of each rank's experts == oracle global kept; send offsets are prefixes of kl
    nl = n // R
    for rank, out, _, _, kloc, so, *_ , gkept in res:
        assert kloc == gkept[rank * nl:(rank + 1) * nl]
        kl_r = np.array(out[0][1])[rank]
        assert so == np.concatenate([[0], np.cumsum(kl_r)[:-1]]).tolist()
    # message sizes: what all ranks send to owner(e) fills exactly the expert's kept slots,
    # contiguously (rank r's block starts at pre[r][e]) and never beyond the capacity
    pre_a, kl_a = np.array(plans[0][0][0]), np.array(plans[0][0][1])
    gkept = res[0][-1]
    for e in range(n):
        assert kl_a[:, e].sum() == gkept[e] <= cap[e]
        for r in range(R):
            if kl_a[r, e]:
                assert pre_a[r, e] + kl_a[r, e] <= cap[e]
                assert pre_a[r, e] == kl_a[:r, e].sum()       # no gap before rank r's block


class _FakeLayer:
    """Stands in for MoELayer's IPC window calls: rank `bad` cannot open its peers' windows."""

    def __init__(self, rank, bad):
        self.rank, self.bad, self.got = rank, bad, None

    def peer_export(self):
        return bytes([self.rank]) * 64

    def peer_import(self, handles):
        if self.rank == self.bad:
            raise RuntimeError("cudaIpcOpenMemHandle failed")
        self.got = [h[0] for h in handles]


def _connect_worker(rank, R, port, bad, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=R)
    from paper_2205_01848_b200.dist import peer_connect
    L = _FakeLayer(rank, bad)
    ok = peer_connect(L, strict=False)
    try:
        peer_connect(_FakeLayer(rank, bad), strict=True)
        strict_raised = False
    except RuntimeError:
        strict_raised = True
    q.put((rank, ok, strict_raised, L.got))
    dist.destroy_process_group()


@pytest.mark.parametrize("bad", [-1, 1])
def test_peer_connect_ranks_agree(bad):
    """Every rank learns whether EVERY rank opened the windows (bench.py then switches all
    ranks to the NCCL transport together instead of hanging or diverging)."""
    R = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_connect_worker, args=(r, R, port, bad, q)) for r in range(R)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(R))
    for p in ps:
        p.join(timeout=60)
    for rank, ok, strict_raised, got in res:
        assert ok == (bad < 0) and strict_raised == (bad >= 0)
        if rank != bad:
            assert got == list(range(R))
