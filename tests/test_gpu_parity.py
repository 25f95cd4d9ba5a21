"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by element.

Routing (idx, fresh idx, slot_of, token_of_slot, counts, kept, drops, hit_count) must be
bit-exact given the GPU's fp32 logits; values within 1e-5 (fp32) / 2e-2 (bf16) relative
(||a-b||_inf/||b||_inf), per the north star.
"""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from synth import perturb_cached

from parity_util import (assert_routing_exact, assert_values, checked_relu_mask, kernel_relu_mask,
                         rel, run_pair)

pytestmark = pytest.mark.gpu


def _caps(n, T, k, alpha):
    return O.capacities_from_factors([alpha] * n, T, k)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,k", [(4, 1), (4, 2), (8, 2), (16, 1)])
@pytest.mark.parametrize("renorm", [0, 1])
def test_layer_parity_small(dtype, n, k, renorm):
    T, d, f = 1000, 64, 128          # 8 routing tiles with a ragged tail (1000 = 7*128 + 104)
    caps = _caps(n, T, k, 1.0)       # alpha = 1: drops happen
    layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, dtype, caps, renorm)
    assert st.routing.drops > 0
    assert_routing_exact(gpu, st, k)
    assert_values(gpu, st, gr, ol, dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layer_parity_wide(dtype):
    n, k, T, d, f, do = 32, 2, 700, 128, 320 if dtype == "f32" else 256, 192
    caps = _caps(n, T, k, 1.25)
    layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, dtype, caps, 1, d_out=do)
    assert_routing_exact(gpu, st, k)
    assert_values(gpu, st, gr, ol, dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_ties_regime_exact_routing(dtype):
    # integer logits: top-k ties everywhere; lower expert index must win (reading 3)
    n, k, T, d, f = 8, 2, 513, 64, 64
    caps = _caps(n, T, k, 1.0)
    layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, dtype, caps, 1, regime="ties")
    lg = gpu["routing_fwd"]["logits"]
    assert np.array_equal(lg, np.round(lg))            # exact integers on the GPU
    ties = sum(len(set(row.tolist())) < n for row in lg)
    assert ties > T // 2
    assert_routing_exact(gpu, st, k)
    assert_values(gpu, st, gr, ol, dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_skewed_heavy_drops_and_capacity_one(dtype):
    n, k, T, d, f = 16, 1, 900, 64, 128
    for caps in (_caps(n, T, k, 1.0), [1] * n, [T] * n):
        layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, dtype, caps, 0, regime="skewed")
        assert_routing_exact(gpu, st, k)
        assert_values(gpu, st, gr, ol, dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_k_equals_n_dense_mixture(dtype):
    n = k = 4
    T, d, f = 300, 64, 64
    layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, dtype, [T] * n, 1)
    assert st.routing.drops == 0
    assert_routing_exact(gpu, st, k)
    assert_values(gpu, st, gr, ol, dtype)


def test_empty_batch():
    from paper_2205_01848_b200 import MoELayer
    layer = MoELayer(4, 2, 64, 64, 0, 128, "f32", 1, device="cuda")
    x = torch.empty(0, 64, device="cuda")
    p = dict(w_gate=torch.randn(4, 64, device="cuda"), w1=torch.randn(4, 64, 64, device="cuda"),
             b1=torch.randn(4, 64, device="cuda"), w2=torch.randn(4, 64, 64, device="cuda"),
             b2=torch.randn(4, 64, device="cuda"))
    y = layer.forward(x, p["w_gate"], p["w1"], p["b1"], p["w2"], p["b2"])
    g = layer.backward(torch.empty(0, 64, device="cuda"))
    torch.cuda.synchronize()
    assert y.shape == (0, 64)
    assert float(g["dw1"].abs().max()) == 0.0 and float(g["dw_gate"].abs().max()) == 0.0
    assert layer.stats()["counts"] == [0, 0, 0, 0]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_cached_assignment(dtype):
    n, k, T, d, f = 16, 2, 800, 64, 128
    caps = _caps(n, T, k, 1.25)
    # cache-converged regime: 3 % of rows stale
    layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, dtype, caps, 1,
                                      cached=lambda fresh: perturb_cached(fresh, n, 0.03))
    assert 0 < st.hit_count < T
    assert_routing_exact(gpu, st, k)
    assert_values(gpu, st, gr, ol, dtype)
    # cached == fresh -> identical to the uncached layer
    layer2, gpu2, st2, gr2, ol2 = run_pair(n, k, d, f, T, dtype, caps, 1,
                                           cached=lambda fresh: fresh)
    layer3, gpu3, st3, gr3, ol3 = run_pair(n, k, d, f, T, dtype, caps, 1)
    assert gpu2["stats"]["hit_count"] == T
    for key in ("y", "dx", "dw1", "dw_gate"):
        assert np.array_equal(gpu2[key], gpu3[key]), key


def test_invalid_cached_index_flag():
    from paper_2205_01848_b200 import MoELayer
    from paper_2205_01848_b200._lib import MOE_ERR_DEVICE_FLAG
    n, k, T, d = 4, 2, 64, 64
    layer = MoELayer(n, k, d, d, 0, T, "f32", 1, device="cuda")
    bad = torch.zeros(T, k, dtype=torch.int32, device="cuda")     # duplicate experts
    layer.set_cached_assignment(bad)
    x = torch.randn(T, d, device="cuda")
    p = [torch.randn(n, d, device="cuda"), torch.randn(n, d, d, device="cuda"),
         torch.randn(n, d, device="cuda"), torch.randn(n, d, d, device="cuda"),
         torch.randn(n, d, device="cuda")]
    layer.forward(x, *p)
    st, fl = layer.check_flags()
    assert st == MOE_ERR_DEVICE_FLAG and fl & 2
    assert layer.check_flags() == (0, 0)           # flags cleared after report


def test_nan_logit_flag():
    from paper_2205_01848_b200 import MoELayer
    n, k, T, d = 4, 1, 64, 64
    layer = MoELayer(n, k, d, d, 0, T, "f32", 1, device="cuda")
    x = torch.randn(T, d, device="cuda")
    x[3, 5] = float("nan")
    p = [torch.randn(n, d, device="cuda"), torch.randn(n, d, d, device="cuda"),
         torch.randn(n, d, device="cuda"), torch.randn(n, d, d, device="cuda"),
         torch.randn(n, d, device="cuda")]
    layer.forward(x, *p)
    st, fl = layer.check_flags()
    assert fl & 1


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_recompile_capacities(dtype):
    """Dynamic capacity (S4.1): changing capacities is stream-ordered, preserves weights,
    and with no drops on either side gives bitwise-identical outputs."""
    from paper_2205_01848_b200 import MoELayer
    from synth import make_layer
    n, k, T, d, f = 8, 2, 640, 64, 128
    cpu = make_layer(n, d, f, d, T, dtype)
    g = {kk: v.cuda() for kk, v in cpu.items()}
    snap = {kk: v.clone() for kk, v in g.items()}
    layer = MoELayer(n, k, d, f, 0, T, dtype, 1, device="cuda")
    layer.set_capacities([T] * n)
    y1 = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"]).clone()
    counts = layer.stats()["counts"]
    layer.set_capacities([max(1, c) for c in counts])  # tight: still no drops
    y2 = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"]).clone()
    assert layer.stats()["drops"] == 0
    layer.set_capacities([max(1, c // 2) for c in counts])   # shrink: drops appear
    y3 = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"]).clone()
    st3 = layer.stats()
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert st3["drops"] == sum(max(0, c - max(1, c // 2)) for c in counts)
    assert not torch.equal(y1, y3)
    for kk in snap:
        assert torch.equal(snap[kk], g[kk]), f"{kk} modified"


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_determinism(dtype):
    n, k, T, d, f = 16, 2, 900, 64, 128
    caps = _caps(n, T, k, 1.0)
    _, a, _, _, _ = run_pair(n, k, d, f, T, dtype, caps, 0)
    _, b, _, _, _ = run_pair(n, k, d, f, T, dtype, caps, 0)
    for key in ("y", "dx", "dw_gate", "dw1", "db1", "dw2", "db2"):
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("dtype,k,d,f,renorm,fusion", [
    ("f32", 2, 64, 64, 1, 0),
    ("bf16", 1, 128, 256, 0, 6),   # fused dispatch backward (+ drop-only pass) accumulating
    ("bf16", 2, 128, 256, 1, 0),   # 2-CTA GEMMs, db1 from DGRAD_A, unfused gate-dx
    ("bf16", 1, 128, 256, 0, 14),  # default flags: + O in token order
    ("bf16", 2, 128, 256, 1, 8),   # k = 2, O in token order (separate combine)
])
def test_accumulate_gradients(dtype, k, d, f, renorm, fusion):
    n, T = 8, 520
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    from synth import make_dy, make_layer
    cpu = make_layer(n, d, f, d, T, dtype)
    g = {kk: v.cuda() for kk, v in cpu.items()}
    dy = make_dy(T, d, dtype).cuda()
    layer = MoELayer(n, k, d, f, 0, T, dtype, renorm, device="cuda")
    layer.set_fusion(fusion)
    layer.set_capacities(capacity_from_factors([0.8] * n, T, k))   # with drops
    layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    g1 = layer.backward(dy)
    acc = {kk: v.clone() for kk, v in g1.items()}
    layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    layer.backward(dy, grads=acc, accumulate=True)
    torch.cuda.synchronize()
    tol = 1e-6 if dtype == "f32" else 1e-2
    for kk in g1:
        a, b = acc[kk].float(), 2 * g1[kk].float()
        assert (a - b).abs().max().item() <= tol * max(b.abs().max().item(), 1e-30), kk


def test_backward_without_forward_is_state_error():
    from paper_2205_01848_b200 import MoELayer, MoEError
    layer = MoELayer(4, 1, 64, 64, 0, 64, "f32", 1, device="cuda")
    layer._saved = (torch.zeros(1, 64, device="cuda"),) * 6
    with pytest.raises(MoEError):
        layer.backward(torch.zeros(1, 64, device="cuda"))


def test_autograd_function_matches_layer():
    from paper_2205_01848_b200 import DynaMoE
    torch.manual_seed(0)
    m = DynaMoE(8, 2, 64, 128, 0, 256, "f32", device="cuda")
    x = torch.randn(256, 64, device="cuda", requires_grad=True)
    y = m(x)
    y.square().sum().backward()
    assert x.grad is not None and m.w1.grad is not None and m.w_gate.grad is not None
    assert torch.isfinite(x.grad).all()


@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("k,renorm", [(1, 0), (2, 1)])
def test_multitile_stress_bf16(k, renorm):
    """More tiles than SM pairs in every tcgen05 GEMM (persistent loops wrap, multi-k-block
    weight-gradient tiles, fused bias warps): guards the pipeline/barrier protocols."""
    n, T, d, f = 64, 8192, 256, 1024
    caps = _caps(n, T, k, 1.0)
    layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, "bf16", caps, renorm)
    assert_routing_exact(gpu, st, k)
    assert_values(gpu, st, gr, ol, "bf16")


@pytest.mark.parametrize("k,renorm", [(2, 1), (1, 0), (2, 0)])
def test_confident_router_dl_precision(k, renorm):
    """A near one-hot router (W_g scaled x25: the top probability is ~1): dl is a tiny
    difference of the experts' dw, and the cancellation-free closed forms keep it within the
    fp32 budget of the oracle (the plain w_r (dw_r - sum w dw) loses ~5 digits here)."""
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    from synth import make_dy, make_layer, to_numpy64
    n, d, f, T = 8, 64, 128, 600
    cpu = make_layer(n, d, f, d, T, "f32")
    cpu["w_gate"] = cpu["w_gate"] * 25.0
    dy = make_dy(T, d, "f32")
    caps = capacity_from_factors([4.0] * n, T, k)
    layer = MoELayer(n, k, d, f, 0, T, "f32", renorm, device="cuda")
    layer.set_capacities(caps)
    g = {kk: v.cuda() for kk, v in cpu.items()}
    layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    rt = layer.routing(T)
    grads = layer.backward(dy.cuda())
    torch.cuda.synchronize()
    p64 = {kk: to_numpy64(v) for kk, v in cpu.items() if kk != "x"}
    st = O.moe_forward(to_numpy64(cpu["x"]), p64, k, caps, renorm,
                       logits=rt["logits"].cpu().double().numpy())
    mask = checked_relu_mask(st, kernel_relu_mask(rt, st), "confident router")
    gr = O.moe_backward(st, to_numpy64(dy), relu_mask=mask)
    assert float(np.max(st.p)) > 0.999999   # the regime this test is about
    dl = layer.routing(T)["dl"].cpu().double().numpy()
    assert rel(dl, gr["dl"]) <= 1e-5
    assert rel(to_numpy64(grads["dw_gate"]), gr["dw_gate"]) <= 1e-5


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_maximum_experts_and_topk(dtype):
    """The largest configuration the library accepts (n = 256 experts, the capacity table's
    size; k = 8, MOE_MAX_K) against the oracle, with drops; one expert more or one choice
    more is refused at moe_init."""
    n, k, T, d, f = 256, 8, 600, 64, 64
    caps = _caps(n, T, k, 1.0)
    layer, gpu, st, gr, ol = run_pair(n, k, d, f, T, dtype, caps, 1)
    assert st.routing.drops > 0
    assert_routing_exact(gpu, st, k)
    assert_values(gpu, st, gr, ol, dtype)
    from paper_2205_01848_b200 import MoELayer
    for nn, kk in ((257, 1), (16, 9)):
        with pytest.raises(Exception):
            MoELayer(nn, kk, d, f, 0, T, dtype, 1, device="cuda")
