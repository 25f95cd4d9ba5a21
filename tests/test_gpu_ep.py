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


def _run_virtual(R, n, k, T, d, f, dtype, renorm, cached_frac=None, lam=0.0, transport="nccl",
                 iters=1, caps_seq=None, fusion=0, keep_h=False):
    """R expert-parallel ranks as threads on one GPU -- over the library's virtual NCCL-style
    communicator, or through the peer-memory transport (N1) with in-process windows -- against
    the single-GPU layer on the concatenated batch.  iters > 1 repeats forward+backward
    (caps_seq[i] = capacities of iteration i), returning the last iteration."""
    import ctypes as C
    import threading
    from paper_2205_01848_b200 import MoELayer, _lib
    from paper_2205_01848_b200.dist import peer_connect_local
    from synth import make_dy, make_layer
    lib = _lib.load()
    comm = C.c_void_p()
    if transport == "nccl":
        assert lib.moe_vcomm_create(R, C.byref(comm)) == 0
    Tg = R * T
    cpu = make_layer(n, d, f, d, Tg, dtype)
    g = {kk: v.cuda() for kk, v in cpu.items()}
    dy = make_dy(Tg, d, dtype).cuda()
    caps = O.capacities_from_factors([1.0] * n, Tg, k)
    if caps_seq is None:
        caps_seq = [caps] * iters
    caps = caps_seq[-1]
    cached = None
    if cached_frac is not None:
        from synth import perturb_cached
        fresh = O.topk_sorted(O.gate_logits(to_np(cpu["x"]), to_np(cpu["w_gate"])), k)
        cached = torch.from_numpy(perturb_cached(fresh, n, cached_frac)).cuda()
    if transport == "peer":
        # Load every kernel this shape uses before the threaded ranks run: with CUDA lazy
        # loading, a rank spinning in a barrier kernel while another thread's first launch
        # loads a module can stall until the barrier's bounded wait gives up (one process,
        # one GPU; separate processes per GPU are not affected).
        warm = MoELayer(n, k, d, f, 0, T, dtype, renorm, world_size=1, rank=0, device="cuda",
                        transport="peer")
        warm.peer_attach([warm.peer_window()])
        warm.set_balance_loss(lam)
        warm.forward(g["x"][:T], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
        warm.backward(dy[:T].contiguous())
        torch.cuda.synchronize()
        warm.close()
    layers = [MoELayer(n, k, d, f, 0, T, dtype, renorm, world_size=R, rank=r,
                       nccl_comm=comm.value or 0, device="cuda", transport=transport)
              for r in range(R)]
    if transport == "peer":
        peer_connect_local(layers)
    out = [None] * R
    errs = []

    def work(r):
        try:
            L = layers[r]
            L.set_fusion(fusion)
            L.set_balance_loss(lam)
            if cached is not None:
                L.set_cached_assignment(cached[r * T:(r + 1) * T].contiguous())
            s = torch.cuda.Stream()
            for it in range(iters):
                L.set_capacities(caps_seq[it])
                with torch.cuda.stream(s):
                    xs = g["x"][r * T:(r + 1) * T]
                    y = L.forward(xs, g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
                    hs = L.h_snapshot() if keep_h else None
                    gr = L.backward(dy[r * T:(r + 1) * T].contiguous())
            with torch.cuda.stream(s):
                s.synchronize()
                rt = L.routing(T)
                s.synchronize()
            if hs is not None:
                rt["h_fwd"], rt["h_base"] = hs
            out[r] = (y, gr, rt, L.stats())
        except Exception as ex:  # surfaced in the main thread
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    ref = MoELayer(n, k, d, f, 0, Tg, dtype, renorm, device="cuda")
    # the N2 flags the ranks actually apply (the dx fusion rounds dX + dl W_g once): the peer
    # transport fuses the dispatch backward into the owners' dX GEMMs, the NCCL-style
    # transport does not (its dX rows travel back unfused)
    ref.set_fusion(fusion if transport == "peer" else fusion & ~4)
    ref.set_capacities(caps)
    ref.set_balance_loss(lam)
    if cached is not None:
        ref.set_cached_assignment(cached)
    y_ref = ref.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    st_ref = ref.stats()
    gr_ref = ref.backward(dy)
    rt_ref = ref.routing(Tg)
    torch.cuda.synchronize()
    if transport == "nccl":
        lib.moe_vcomm_destroy(comm)
    for L in layers:
        L.close()
    return out, (y_ref, gr_ref, rt_ref, st_ref)


def to_np(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("R", [2, 4])
@pytest.mark.parametrize("dtype,k,renorm", [("bf16", 2, 1), ("bf16", 1, 0), ("f32", 2, 0)])
def test_ep_virtual_ranks_match_single_gpu(R, dtype, k, renorm):
    n, T, d, f = 16, 512, 64, 128
    out, (y_ref, gr_ref, rt_ref, st_ref) = _run_virtual(R, n, k, T, d, f, dtype, renorm)
    nl = n // R
    # routing: global slots, counts and drops are independent of R (reading 12)
    assert np.array_equal(np.concatenate([o[2]["slot_of"].cpu().numpy() for o in out]),
                          rt_ref["slot_of"].cpu().numpy())
    for o in out:
        assert o[3]["counts"] == st_ref["counts"] and o[3]["drops"] == st_ref["drops"]
    # token-side outputs bit-identical; expert gradients of each rank's experts bit-identical
    assert torch.equal(torch.cat([o[0] for o in out]), y_ref)
    assert torch.equal(torch.cat([o[1]["dx"] for o in out]), gr_ref["dx"])
    for r, o in enumerate(out):
        sl = slice(r * nl, (r + 1) * nl)
        for key in ("dw1", "db1", "dw2", "db2"):
            assert torch.equal(o[1][key][sl], gr_ref[key][sl]), (r, key)
        # dW_g: per-rank partials all-reduced in fp32 (a different summation split)
        a, b = to_np(o[1]["dw_gate"]), to_np(gr_ref["dw_gate"])
        assert np.abs(a - b).max() <= (1e-5 if dtype == "f32" else 1e-2) * np.abs(b).max()


@pytest.mark.timeout(300, method="thread")
def test_ep_virtual_ranks_cached_and_balance():
    n, T, d, f, R = 16, 512, 64, 128, 2
    out, (y_ref, gr_ref, rt_ref, st_ref) = _run_virtual(R, n, 2, T, d, f, "bf16", 1,
                                                        cached_frac=0.03, lam=0.2)
    assert torch.equal(torch.cat([o[0] for o in out]), y_ref)
    assert sum(o[3]["hit_count"] for o in out) == st_ref["hit_count"]
    assert np.allclose(np.concatenate([o[2]["dl"].cpu().numpy() for o in out]),
                       rt_ref["dl"].cpu().numpy(), rtol=1e-5, atol=1e-7)


# --------------------------------------------------------------------------------------
# Peer-memory transport: device-initiated exchange, no host sync
# --------------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,k,renorm", [(8, 2, 1), (16, 1, 0)])
def test_peer_loopback_parity(dtype, n, k, renorm):
    """R = 1 through the peer path (plan kernel, window buffers, barriers, rank-order sums)."""
    from paper_2205_01848_b200 import MoELayer
    T, d, f = 1000, 64, 128
    caps = O.capacities_from_factors([1.0] * n, T, k)
    pl = MoELayer(n, k, d, f, 0, T, dtype, renorm, world_size=1, rank=0, device="cuda",
                  transport="peer")
    pl.peer_attach([pl.peer_window()])
    layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, dtype, caps, renorm, layer=pl)
    assert st.routing.drops > 0
    assert_routing_exact(gpu, st, k, check_token_of_slot=True)
    assert_values(gpu, st, gr, ol, dtype)
    _, ref, _, _, _ = run_pair(n, k, d, f, T, dtype, caps, renorm)
    for key in ("y", "dx", "dw1", "db1", "dw2", "db2", "dw_gate"):
        assert np.array_equal(gpu[key], ref[key]), key


def _check_virtual(out, ref, R, n, dtype):
    y_ref, gr_ref, rt_ref, st_ref = ref
    nl = n // R
    assert np.array_equal(np.concatenate([o[2]["slot_of"].cpu().numpy() for o in out]),
                          rt_ref["slot_of"].cpu().numpy())
    for o in out:
        assert o[3]["counts"] == st_ref["counts"] and o[3]["drops"] == st_ref["drops"]
    assert torch.equal(torch.cat([o[0] for o in out]), y_ref)
    assert torch.equal(torch.cat([o[1]["dx"] for o in out]), gr_ref["dx"])
    for r, o in enumerate(out):
        sl = slice(r * nl, (r + 1) * nl)
        for key in ("dw1", "db1", "dw2", "db2"):
            assert torch.equal(o[1][key][sl], gr_ref[key][sl]), (r, key)
            # the other ranks' expert slices are zeroed by the library (moe.h), not garbage
            other = torch.ones(n, dtype=torch.bool)
            other[sl] = False
            assert not o[1][key][other.cuda()].any(), (r, key, "non-local slice not zero")
        a, b = to_np(o[1]["dw_gate"]), to_np(gr_ref["dw_gate"])
        assert np.abs(a - b).max() <= (1e-5 if dtype == "f32" else 1e-2) * np.abs(b).max()


@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("R", [2, 4])
@pytest.mark.parametrize("dtype,k,renorm", [("bf16", 2, 1), ("bf16", 1, 0), ("f32", 2, 0)])
def test_peer_virtual_ranks_match_single_gpu(R, dtype, k, renorm):
    n, T, d, f = 16, 512, 64, 128
    out, ref = _run_virtual(R, n, k, T, d, f, dtype, renorm, transport="peer")
    _check_virtual(out, ref, R, n, dtype)
    # dW_g is summed in rank order from the windows: identical on every rank
    for o in out[1:]:
        assert torch.equal(o[1]["dw_gate"], out[0][1]["dw_gate"])
    # each owner's token_of_slot holds the global token ids of its experts' kept rows,
    # exactly the single-GPU table (reading 12)
    rt_ref = ref[2]
    nl = n // R
    kept = [min(c, cap) for c, cap in zip(ref[3]["counts"],
                                          O.capacities_from_factors([1.0] * n, R * T, k))]
    for r, o in enumerate(out):
        rt = o[2]
        for j in range(nl):
            e = r * nl + j
            a = rt["token_of_slot"][rt["base"][j]: rt["base"][j] + kept[e]].cpu().numpy()
            b0 = rt_ref["base"][e]
            b = rt_ref["token_of_slot"][b0: b0 + kept[e]].cpu().numpy()
            assert np.array_equal(a, b), (r, e)


@pytest.mark.timeout(300, method="thread")
def test_peer_virtual_ranks_cached_and_balance():
    n, T, d, f, R = 16, 512, 64, 128, 2
    out, (y_ref, gr_ref, rt_ref, st_ref) = _run_virtual(R, n, 2, T, d, f, "bf16", 1,
                                                        cached_frac=0.03, lam=0.2,
                                                        transport="peer")
    assert torch.equal(torch.cat([o[0] for o in out]), y_ref)
    assert sum(o[3]["hit_count"] for o in out) == st_ref["hit_count"]
    assert np.allclose(np.concatenate([o[2]["dl"].cpu().numpy() for o in out]),
                       rt_ref["dl"].cpu().numpy(), rtol=1e-5, atol=1e-7)


@pytest.mark.timeout(300, method="thread")
def test_peer_virtual_ranks_many_iterations_with_recompiles():
    """Barrier epochs advance in lockstep over iterations; capacity changes (recompiles)
    between iterations re-lay out every owner's regions."""
    n, T, d, f, R, k = 16, 384, 64, 128, 4, 2
    Tg = R * T
    seq = [O.capacities_from_factors([a] * n, Tg, k) for a in (1.0, 0.5, 2.0, 1.25, 0.75)]
    out, ref = _run_virtual(R, n, k, T, d, f, "bf16", 1, transport="peer", iters=len(seq),
                            caps_seq=seq)
    _check_virtual(out, ref, R, n, "bf16")


@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("fusion", [0, 6])
@pytest.mark.parametrize("R", [2, 4])
@pytest.mark.parametrize("k,renorm", [(1, 0), (2, 1)])
def test_peer_return_rows_virtual_ranks(R, k, renorm, fusion):
    """N1 return rows: with d, d_out multiples of 128 the owners' FWD2 / DGRAD_X epilogues
    store O / dX rows straight into the token owners' windows in (token, choice) order, and
    the combine / gate-dx kernels read them locally -- bitwise equal to the single-GPU layer
    and to the owner-read form (MOE_PEER_RET=0).  fusion 6 with k = 1: the owners' dX GEMMs
    also add dl W_g (pairs pushed by the token owners' combine backward) and return dx rows
    -- bitwise equal to the single-GPU fused dispatch backward."""
    import os
    n, T, d, f = 16, 512, 128, 256
    out, ref = _run_virtual(R, n, k, T, d, f, "bf16", renorm, transport="peer", fusion=fusion)
    _check_virtual(out, ref, R, n, "bf16")
    for o in out[1:]:
        assert torch.equal(o[1]["dw_gate"], out[0][1]["dw_gate"])
    if fusion:
        return  # the owner-read form has no fused dispatch backward (compared at fusion 0)
    os.environ["MOE_PEER_RET"] = "0"
    try:
        out0, _ = _run_virtual(R, n, k, T, d, f, "bf16", renorm, transport="peer")
    finally:
        del os.environ["MOE_PEER_RET"]
    nl = n // R
    for r, (a, b) in enumerate(zip(out, out0)):
        assert torch.equal(a[0], b[0])
        for key in ("dx", "dw_gate"):
            assert torch.equal(a[1][key], b[1][key]), key
        for key in ("dw1", "db1", "dw2", "db2"):  # each rank writes its own experts only
            sl = slice(r * nl, (r + 1) * nl)
            assert torch.equal(a[1][key][sl], b[1][key][sl]), key


@pytest.mark.parametrize("k,renorm", [(1, 0), (2, 1)])
def test_peer_return_rows_loopback_oracle(k, renorm):
    """R = 1 peer path with return rows (d = 128) against the oracle."""
    from paper_2205_01848_b200 import MoELayer
    n, T, d, f = 16, 1000, 128, 256
    caps = O.capacities_from_factors([1.0] * n, T, k)
    pl = MoELayer(n, k, d, f, 0, T, "bf16", renorm, world_size=1, rank=0, device="cuda",
                  transport="peer")
    pl.peer_attach([pl.peer_window()])
    layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, "bf16", caps, renorm, layer=pl)
    assert st.routing.drops > 0
    assert_routing_exact(gpu, st, k, check_token_of_slot=True)
    assert_values(gpu, st, gr, ol, "bf16")


@pytest.mark.parametrize("dtype,n,k,renorm", [("bf16", 16, 1, 0), ("f32", 8, 2, 1)])
def test_peer_windows_on_nccl_symmetric_memory(comm, dtype, n, k, renorm):
    """N1 on NCCL's symmetric memory: the peer window is re-allocated with ncclMemAlloc,
    registered on torch's communicator (ncclCommWindowRegister, SYMMETRIC) and mapped through
    the NCCL device API (ncclGetPeerPointer, LSA team); the layer then matches the oracle and
    the single-GPU path bit for bit (1-rank loopback: one GPU here)."""
    from paper_2205_01848_b200 import MoELayer
    T, d, f = 777, 128, 256
    caps = O.capacities_from_factors([1.0] * n, T, k)
    pl = MoELayer(n, k, d, f, 0, T, dtype, renorm, world_size=1, rank=0, device="cuda",
                  transport="peer")
    pl.peer_connect_nccl(comm)
    assert pl.peer_via == "nccl-symmetric-window"
    try:
        layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, dtype, caps, renorm, layer=pl)
        assert st.routing.drops > 0
        assert_routing_exact(gpu, st, k, check_token_of_slot=True)
        assert_values(gpu, st, gr, ol, dtype)
        _, ref, _, _, _ = run_pair(n, k, d, f, T, dtype, caps, renorm)
        for key in ("y", "dx", "dw1", "db1", "dw2", "db2", "dw_gate"):
            assert np.array_equal(gpu[key], ref[key]), key
        assert layer.check_flags()[1] == 0
    finally:
        pl.close()   # deregisters the window while the communicator is alive


@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("R", [2, 4])
@pytest.mark.parametrize("dtype,k,renorm", [("bf16", 2, 1), ("bf16", 1, 0), ("f32", 2, 0)])
def test_peer_virtual_ranks_vs_oracle(R, dtype, k, renorm):
    """R > 1 expert-parallel ranks (peer transport) against the fp64 oracle DIRECTLY, not only
    against the single-GPU layer: the oracle runs the concatenated global batch with the
    ranks' fp32 logits (routing decisions, reading 3) and global capacities (reading 12);
    y / dx / dl / dw per token from the token owners, dW1 / db1 / dW2 / db2 from each expert's
    owner, dW_g from the rank-order window sum; ReLU' decisions from each owner's stored H
    within the fp32 rounding band (checked_relu_mask)."""
    from parity_util import TOL, checked_relu_mask, rel, rel_rows
    n, T, d, f = 16, 512, 64, 128
    out, _ = _run_virtual(R, n, k, T, d, f, dtype, renorm, transport="peer", keep_h=True)
    from synth import make_dy, make_layer, to_numpy64
    Tg, nl = R * T, n // R
    cpu = make_layer(n, d, f, d, Tg, dtype)
    dy64 = to_numpy64(make_dy(Tg, d, dtype))
    x64 = to_numpy64(cpu["x"])
    p64 = {kk: to_numpy64(v) for kk, v in cpu.items() if kk != "x"}
    caps = O.capacities_from_factors([1.0] * n, Tg, k)
    lg = np.concatenate([o[2]["logits"].cpu().double().numpy() for o in out])
    st = O.moe_forward(x64, p64, k, caps, renorm, logits=lg, emulate_bf16=(dtype == "bf16"))
    assert st.routing.drops > 0
    assert np.array_equal(np.concatenate([o[2]["slot_of"].cpu().numpy() for o in out]),
                          st.routing.slot_of)
    kmask = []
    for e in range(n):
        rt = out[e // nl][2]
        b = rt["h_base"][e % nl]
        kmask.append((rt["h_fwd"][b: b + int(st.routing.kept[e])].float() > 0).cpu().numpy())
    gr = O.moe_backward(st, dy64, relu_mask=checked_relu_mask(st, kmask, f"R={R}"))
    got = dict(
        y=torch.cat([o[0] for o in out]), dx=torch.cat([o[1]["dx"] for o in out]),
        dw_gate=out[0][1]["dw_gate"],
        **{kk: sum(o[1][kk].float() for o in out) for kk in ("dw1", "db1", "dw2", "db2")})
    got = {kk: to_numpy64(v) for kk, v in got.items()}
    tol = TOL[dtype]
    errs = {"y": rel(got["y"], st.y), "w": rel(np.concatenate([o[2]["w"].cpu().numpy()
                                                               for o in out]), st.w)}
    for kk in ("dx", "dw_gate", "dw1", "db1", "dw2", "db2"):
        errs[kk] = rel(got[kk], gr[kk])
    for kk in ("dw1", "db1", "dw2", "db2"):
        errs[kk + "/expert"] = rel_rows(got[kk], gr[kk])
    errs["dw"] = rel(np.concatenate([o[2]["dw"].cpu().numpy() for o in out]), gr["dw"])
    lim = {kk: (1e-5 if kk == "w" else tol) for kk in errs}
    bad = {kk: v for kk, v in errs.items() if not v <= lim[kk]}
    assert not bad, f"R={R} parity failures {bad} (all: {errs})"
