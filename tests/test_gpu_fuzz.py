"""Seeded sweep of layer shapes x routing regimes x fusion flags against the fp64 oracle
(routing bit-exact, values within the dtype budget).  Shapes are drawn to hit the kernel
variants: 1-CTA and 2-CTA tcgen05 GEMMs (BN 128 / 256), n not a multiple of 64, k up to 8,
d_out != d, ragged T (including T < one routing tile), capacity factors from heavy drops to
none, every N2 fusion flag."""
import numpy as np
import pytest

from parity_util import (assert_routing_exact, assert_values, checked_relu_mask, kernel_relu_mask,
                         run_pair)

pytestmark = pytest.mark.gpu


def _cases():
    rng = np.random.default_rng(2205)
    out = []
    for i in range(160):
        dtype = "bf16" if i % 3 else "f32"
        n = int(rng.choice([3, 8, 16, 40, 64, 130]))
        k = int(min(n, rng.choice([1, 1, 2, 2, 4, 8])))
        d = int(rng.choice([64, 128, 192, 256]))
        f = int(rng.choice([64, 128, 256, 384, 512]))
        d_out = int(rng.choice([0, 0, 128, 64]))
        T = int(rng.choice([1, 5, 127, 300, 777, 1500]))
        alpha = float(rng.choice([0.25, 0.5, 1.0, 1.25, 2.0, 7.0]))
        renorm = int(rng.integers(0, 2))
        regime = str(rng.choice(["uniform", "skewed", "ties"]))
        fusion = int(rng.choice([0, 2, 4, 14, 15]))
        out.append((dtype, n, k, d, f, d_out, T, alpha, renorm, regime, fusion))
    return out


@pytest.mark.parametrize("dtype,n,k,d,f,d_out,T,alpha,renorm,regime,fusion", _cases())
def test_fuzz_vs_oracle(dtype, n, k, d, f, d_out, T, alpha, renorm, regime, fusion):
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    caps = capacity_from_factors([alpha] * n, T, k)
    layer = MoELayer(n, k, d, f, d_out, T, dtype, renorm, device="cuda")
    layer.set_fusion(fusion)
    layer, gpu, st, gr, own = run_pair(n, k, d, f, T, dtype, caps, renorm=renorm, regime=regime,
                                       d_out=d_out or None, layer=layer)
    assert_routing_exact(gpu, st, k)
    assert_values(gpu, st, gr, own, dtype)


def _ep_cases():
    rng = np.random.default_rng(1848)
    out = []
    for i in range(30):
        R = int(rng.choice([2, 4]))
        n = R * int(rng.choice([1, 2, 4, 8]))
        k = int(min(n, rng.choice([1, 2, 2, 4])))
        dtype = "f32" if i % 4 == 0 else "bf16"
        d = int(rng.choice([64, 128, 192]))
        f = int(rng.choice([64, 128, 256]))
        T = int(rng.choice([64, 200, 512]))
        renorm = int(rng.integers(0, 2))
        transport = str(rng.choice(["peer", "nccl"]))
        out.append((R, n, k, dtype, d, f, T, renorm, transport))
    return out


@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("R,n,k,dtype,d,f,T,renorm,transport", _ep_cases())
def test_fuzz_ep_virtual_ranks(R, n, k, dtype, d, f, T, renorm, transport):
    """R expert-parallel ranks (threads on one GPU; peer windows or the virtual communicator)
    against the single-GPU layer on the concatenated batch: routing, y, dx and each owner's
    expert gradients bitwise equal (dW_g within tolerance: summed in another split)."""
    from test_gpu_ep import _check_virtual, _run_virtual
    out, ref = _run_virtual(R, n, k, T, d, f, dtype, renorm, transport=transport)
    _check_virtual(out, ref, R, n, dtype)


def _feature_cases():
    rng = np.random.default_rng(353)
    out = []
    for i in range(48):
        dtype = "bf16" if i % 4 else "f32"
        n = int(rng.choice([4, 8, 16, 64]))
        k = int(min(n, rng.choice([1, 2, 4])))
        d = int(rng.choice([64, 128, 256]))
        f = int(rng.choice([128, 256]))
        T = int(rng.choice([33, 256, 700]))
        renorm = int(rng.integers(0, 2))
        cached = float(rng.choice([-1.0, 0.0, 0.03, 0.5]))   # -1: caching off
        lam = float(rng.choice([0.0, 0.0, 0.3]))
        spec = bool(rng.integers(0, 2))
        fusion = int(rng.choice([0, 14, 15]))
        a1, a2 = (float(v) for v in rng.choice([0.5, 1.0, 1.5, 3.0], 2))
        out.append((dtype, n, k, d, f, T, renorm, cached, lam, spec, fusion, a1, a2))
    return out


@pytest.mark.parametrize("dtype,n,k,d,f,T,renorm,cached,lam,spec,fusion,a1,a2", _feature_cases())
def test_fuzz_features_vs_oracle(dtype, n, k, d, f, T, renorm, cached, lam, spec, fusion, a1, a2):
    """Two iterations with a capacity change (recompile) in between, the second backward
    accumulating into the first's gradients, with random combinations of cached assignments
    (stale fraction), the Eq. 3 balance term, AggregateSpec outputs with spec gradients and
    the N2 fusion flags -- against the oracle run twice with the same inputs."""
    import torch
    from oracle import moe_oracle as O
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    from parity_util import TOL, rel
    from synth import make_dy, make_layer, perturb_cached, to_numpy64
    cpu = make_layer(n, d, f, d, T, dtype)
    g = {kk: v.cuda() for kk, v in cpu.items()}
    x64 = to_numpy64(cpu["x"])
    p64 = {kk: to_numpy64(v) for kk, v in cpu.items() if kk != "x"}
    gen = torch.Generator().manual_seed(7)
    dys = [make_dy(T, d, dtype, seed_offset=i) for i in range(2)]
    dspec = torch.randn(T * k, d, generator=gen).to(cpu["x"].dtype) if spec else None
    dw_ext = torch.randn(T, k, generator=gen) if spec else None
    cidx = None
    if cached >= 0:
        fresh = O.topk_sorted(O.gate_logits(x64, p64["w_gate"]), k)
        cidx = np.ascontiguousarray(perturb_cached(fresh, n, cached) if cached > 0 else fresh,
                                    dtype=np.int32)
    layer = MoELayer(n, k, d, f, 0, T, dtype, renorm, device="cuda")
    layer.set_fusion(fusion)
    layer.set_balance_loss(lam)
    if spec:
        layer.enable_spec(True)
        layer.set_spec_grads(dspec.cuda(), dw_ext.cuda())
    if cidx is not None:
        layer.set_cached_assignment(torch.from_numpy(cidx).cuda())
    grads = None
    want = None
    tol = TOL[dtype]
    for it, alpha in enumerate((a1, a2)):
        caps = capacity_from_factors([alpha] * n, T, k)
        layer.set_capacities(caps)
        y = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
        rt = layer.routing(T)
        grads = layer.backward(dys[it].cuda(), grads=grads, accumulate=it > 0)
        torch.cuda.synchronize()
        st = O.moe_forward(x64, p64, k, caps, renorm, cached_idx=cidx,
                           logits=rt["logits"].cpu().double().numpy(),
                           emulate_bf16=(dtype == "bf16"), balance_lambda=lam)
        assert np.array_equal(rt["slot_of"].cpu().numpy(), st.routing.slot_of), it
        assert rel(to_numpy64(y), st.y) <= tol, it
        mask = checked_relu_mask(st, kernel_relu_mask(rt, st), f"iteration {it}")
        gr = O.moe_backward(st, to_numpy64(dys[it]),
                            dspec=to_numpy64(dspec) if spec else None,
                            dw_ext=dw_ext.double().numpy() if spec else None, relu_mask=mask)
        want = gr if want is None else {kk: want[kk] + gr[kk] for kk in
                                        ("dx", "dw_gate", "dw1", "db1", "dw2", "db2")}
    for kk in ("dx", "dw_gate", "dw1", "db1", "dw2", "db2"):
        assert rel(to_numpy64(grads[kk]), want[kk]) <= tol, kk


def _ep_feature_cases():
    rng = np.random.default_rng(2021)
    out = []
    for i in range(12):
        R = int(rng.choice([2, 4]))
        n = R * int(rng.choice([2, 4]))
        k = int(min(n, rng.choice([1, 2])))
        dtype = "f32" if i % 4 == 0 else "bf16"
        d = int(rng.choice([64, 128]))
        f = 2 * d
        T = int(rng.choice([128, 256]))
        renorm = int(rng.integers(0, 2))
        transport = str(rng.choice(["peer", "nccl"]))
        cached = float(rng.choice([-1.0, 0.03]))
        lam = float(rng.choice([0.0, 0.2]))
        fusion = int(rng.choice([0, 6]))
        out.append((R, n, k, dtype, d, f, T, renorm, transport, cached, lam, fusion))
    return out


@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("R,n,k,dtype,d,f,T,renorm,transport,cached,lam,fusion", _ep_feature_cases())
def test_fuzz_ep_features(R, n, k, dtype, d, f, T, renorm, transport, cached, lam, fusion):
    """Expert-parallel ranks with cached assignments, the balance term, N2 flags and three
    iterations with capacity changes (recompiles) in between, bitwise against one GPU."""
    from oracle import moe_oracle as O
    from test_gpu_ep import _check_virtual, _run_virtual
    Tg = R * T
    seq = [O.capacities_from_factors([a] * n, Tg, k) for a in (1.0, 0.5, 1.5)]
    out, ref = _run_virtual(R, n, k, T, d, f, dtype, renorm, transport=transport,
                            cached_frac=(cached if cached >= 0 else None), lam=lam, iters=3,
                            caps_seq=seq, fusion=fusion)
    _check_virtual(out, ref, R, n, dtype)
