"""N2 fusions (moe_set_fusion): the expert GEMMs gather x rows by
token_of_slot with TMA gather4 (no dispatched X buffer; opt-in, flag 1); for k = 1 the second
GEMM's epilogue writes y = w O (no combine pass, flag 2) and the dX GEMM writes
dx = dX + dl W_g (no dispatch-backward pass, flag 4); the second GEMM stores O in (token,
choice) order for the combine and its backward (flag 8); for k = 2 the epilogue that stores a
token's second O row writes y (flag 16).  Checked against the fp64 oracle
(values within the bf16 budget, routing bit-exact) and against the unfused path of the same
library: BITWISE equal for flags 1, 2, 8 and 16 (same products, same accumulation order); for flag 4
every output but dx is bitwise equal and dx agrees within the bf16 budget (one rounding
instead of two) -- including at the bench's full c3 size."""
import numpy as np
import pytest
import torch

from parity_util import assert_routing_exact, assert_values, run_pair

pytestmark = pytest.mark.gpu


def _run(layer, g, dy, fusion, y_fill=None):
    layer.set_fusion(fusion)
    y = None
    if y_fill is not None:   # poison y: every row must be written (dropped tokens -> 0)
        y = torch.full((g["x"].shape[0], layer.d_out), y_fill, dtype=layer.tdtype,
                       device=layer.device)
    y = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"], y=y)
    grads = None
    if y_fill is not None:   # poison every gradient: all rows must be written
        shapes = dict(dx=g["x"].shape, dw_gate=g["w_gate"].shape, dw1=g["w1"].shape,
                      db1=g["b1"].shape, dw2=g["w2"].shape, db2=g["b2"].shape)
        grads = {kk: torch.full(sh, y_fill, dtype=layer.tdtype, device=layer.device)
                 for kk, sh in shapes.items()}
    grads = layer.backward(dy, grads=grads)
    torch.cuda.synchronize()
    return y.clone(), {k: v.clone() for k, v in grads.items()}


def _bitwise(a, b, what):
    assert a.dtype == b.dtype and a.shape == b.shape
    ai = a.view(torch.int16) if a.dtype == torch.bfloat16 else a.view(torch.int32)
    bi = b.view(torch.int16) if b.dtype == torch.bfloat16 else b.view(torch.int32)
    nbad = int((ai != bi).sum())
    assert nbad == 0, f"{what}: {nbad} elements differ between fused and unfused paths"


def _close(a, b, what, tol=2e-2):
    """dx of the fused dispatch backward: one bf16 rounding instead of two (reading 13)."""
    a, b = a.float(), b.float()
    den = b.abs().max().item()
    err = (a - b).abs().max().item() / (den if den > 0 else 1.0)
    assert err <= tol, f"{what}: rel err {err}"
    # and far tighter than the budget in practice: a few bf16 ulps
    assert err <= 1e-2, f"{what}: rel err {err}"


CASES = [  # n, k, d, f, T, renorm, regime, alpha
    (8, 1, 256, 512, 1000, 0, "uniform", 1.0),    # gather + fused combine, drops
    (8, 1, 256, 512, 1001, 1, "uniform", 1.25),   # renorm (w = 1), ragged T
    (8, 2, 256, 384, 777, 1, "uniform", 1.0),     # k = 2: gather only
    (16, 1, 128, 256, 1500, 0, "skewed", 1.0),    # heavy drops: y rows of dropped tokens = 0
    (4, 1, 128, 128, 3, 0, "uniform", 1.0),       # T < 4 (gather rows past T are OOB)
]


@pytest.mark.parametrize("fusion", [2, 3, 4, 7, 8, 14, 15, 30])
@pytest.mark.parametrize("n,k,d,f,T,renorm,regime,alpha", CASES)
def test_fused_vs_oracle(n, k, d, f, T, renorm, regime, alpha, fusion):
    from paper_2205_01848_b200 import capacity_from_factors
    caps = capacity_from_factors([alpha] * n, T, k)
    from paper_2205_01848_b200 import MoELayer
    layer = MoELayer(n, k, d, f, 0, T, "bf16", renorm, device="cuda")
    layer.set_fusion(fusion)
    layer, gpu, st, gr, own = run_pair(n, k, d, f, T, "bf16", caps, renorm=renorm,
                                       regime=regime, layer=layer)
    assert_routing_exact(gpu, st, k)
    assert_values(gpu, st, gr, own, "bf16")
    if regime == "skewed":
        assert st.routing.drops > 0


@pytest.mark.parametrize("n,k,d,f,T,renorm,regime,alpha", CASES)
def test_fused_bitwise_equals_unfused(n, k, d, f, T, renorm, regime, alpha):
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    from synth import make_dy, make_layer
    g = {kk: v.cuda() for kk, v in make_layer(n, d, f, d, T, "bf16", regime).items()}
    dy = make_dy(T, d, "bf16").cuda()
    layer = MoELayer(n, k, d, f, 0, T, "bf16", renorm, device="cuda")
    layer.set_capacities(capacity_from_factors([alpha] * n, T, k))
    y0, g0 = _run(layer, g, dy, 0, y_fill=float("nan"))
    assert not torch.isnan(y0).any()
    # combine, gather, both, dx, gather+combine+dx, O in token order (alone, + combine,
    # default combine+dx+otok, all), k = 2 combine in the second GEMM (alone with otok, default)
    for fusion in (2, 1, 3, 4, 7, 8, 10, 14, 15, 24, 30):
        y1, g1 = _run(layer, g, dy, fusion, y_fill=float("nan"))
        assert not torch.isnan(y1).any()
        _bitwise(y1, y0, f"y (fusion {fusion})")
        for key in g0:
            if key == "dx" and fusion & 4 and k == 1:
                _close(g1[key], g0[key], f"dx (fusion {fusion})")
            else:
                _bitwise(g1[key], g0[key], f"{key} (fusion {fusion})")


def test_fused_cached_mode_bitwise():
    """Cached indices: the gate runs concurrently with the routing / dispatch / first GEMM on
    the other stream and the second GEMM (fused combine) waits for its weights; results
    equal the unfused path bitwise (y poisoned first: every row must be written)."""
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    from synth import make_dy, make_layer
    n, k, d, f, T = 8, 1, 256, 256, 999
    g = {kk: v.cuda() for kk, v in make_layer(n, d, f, d, T, "bf16").items()}
    dy = make_dy(T, d, "bf16").cuda()
    gen = torch.Generator(device="cpu").manual_seed(5)
    cidx = torch.randint(0, n, (T, k), generator=gen, dtype=torch.int32).cuda()
    layer = MoELayer(n, k, d, f, 0, T, "bf16", 0, device="cuda")
    layer.set_capacities(capacity_from_factors([1.0] * n, T, k))
    layer.set_cached_assignment(cidx)
    y0, g0 = _run(layer, g, dy, 0)
    y1, g1 = _run(layer, g, dy, 3, y_fill=float("nan"))
    _bitwise(y1, y0, "y")
    for key in g0:
        _bitwise(g1[key], g0[key], key)
    y1, g1 = _run(layer, g, dy, 7, y_fill=float("nan"))
    _bitwise(y1, y0, "y")
    for key in g0:
        (_close if key == "dx" else _bitwise)(g1[key], g0[key], f"{key} (fusion 7)")


def test_fused_bitwise_at_bench_size():
    """c3 (the bench workload: 64 experts, top-1, d 1024, f 4096, 65,536 tokens, alpha 1) in
    the launch configuration bench.py times: fused == unfused bitwise, and sampled tokens
    of y equal the plain fp32 definition within the bf16 budget."""
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    from synth import make_dy, make_layer
    n, k, d, f, T = 64, 1, 1024, 4096, 65536
    g = make_layer(n, d, f, d, T, "bf16", device="cuda")
    dy = make_dy(T, d, "bf16", device="cuda")
    layer = MoELayer(n, k, d, f, 0, T, "bf16", 0, device="cuda")
    layer.set_capacities(capacity_from_factors([1.0] * n, T, k))
    y0, g0 = _run(layer, g, dy, 0)
    for fusion in (7, 6):   # end with the default (combine + dx) for the sampled check
        y1, g1 = _run(layer, g, dy, fusion, y_fill=float("nan"))
        _bitwise(y1, y0, f"y (fusion {fusion})")
        for key in g0:
            if key == "dx":
                _close(g1[key], g0[key], f"dx (fusion {fusion})")
            else:
                _bitwise(g1[key], g0[key], f"{key} (fusion {fusion})")
    # sampled tokens against the definition (fp32 from the same bf16 inputs)
    r = layer.routing(T)
    idx = r["idx"][:, 0].long()
    slot = r["slot_of"][:, 0].long()
    w = r["w"][:, 0]
    rng = np.random.default_rng(0)
    for t in rng.choice(T, 48, replace=False).tolist():
        if slot[t] < 0:
            assert y1[t].abs().max().item() == 0.0
            continue
        e = int(idx[t])
        xt = g["x"][t].float()
        h = torch.relu(xt @ g["w1"][e].float().T + g["b1"][e].float())
        h = h.bfloat16().float()
        o = (h @ g["w2"][e].float().T + g["b2"][e].float()).bfloat16().float()
        ref = float(w[t]) * o
        err = (y1[t].float() - ref).abs().max() / ref.abs().max()
        assert err < 2e-2, (t, float(err))


@pytest.mark.parametrize("n,T,alpha,cached", [(8, 999, 1.0, False), (16, 1500, 0.7, False),
                                               (8, 640, 1.0, True)])
def test_k2_combine_in_gemm_bitwise(n, T, alpha, cached):
    """k = 2 combine in the second GEMM's epilogue (flag 16): y bitwise equal to the separate
    combine kernel, with drops (alpha < 1: tokens with one or both pairs dropped), y poisoned
    first, two forwards in a row (the per-(token, block) counters must have reset), and in
    cached mode (the second GEMM waits for the gate weights)."""
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    from synth import make_dy, make_layer
    k, d, f = 2, 256, 256
    g = {kk: v.cuda() for kk, v in make_layer(n, d, f, d, T, "bf16").items()}
    dy = make_dy(T, d, "bf16").cuda()
    layer = MoELayer(n, k, d, f, 0, T, "bf16", 1, device="cuda")
    layer.set_capacities(capacity_from_factors([alpha] * n, T, k))
    if cached:
        gen = torch.Generator(device="cpu").manual_seed(7)
        cidx = torch.stack([torch.randperm(n, generator=gen)[:k] for _ in range(T)]).int().cuda()
        layer.set_cached_assignment(cidx)
    y0, g0 = _run(layer, g, dy, 14, y_fill=float("nan"))
    for _ in range(2):
        y1, g1 = _run(layer, g, dy, 30, y_fill=float("nan"))
        assert not torch.isnan(y1).any()
        _bitwise(y1, y0, "y (k = 2 combine in the GEMM)")
        for key in g0:
            _bitwise(g1[key], g0[key], key)


@pytest.mark.parametrize("n,k,d,T,renorm", [(64, 1, 1024, 4096, 0), (16, 2, 256, 1001, 1),
                                             (130, 2, 128, 777, 0)])
def test_combine_bwd_lean_equals_full(n, k, d, T, renorm):
    """The combine backward's lean instantiation (single GPU, no loss-variant inputs: the dy /
    O rows requested before the routing tables) against the full one (selected by passing
    all-zero spec-row / gate-weight gradients, which add exact zeros): every output of the
    backward bitwise equal (dl, dw, dx and all weight gradients)."""
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    from synth import make_dy, make_layer
    g = {kk: v.cuda() for kk, v in make_layer(n, d, 2 * d, d, T, "bf16").items()}
    dy = make_dy(T, d, "bf16").cuda()
    layer = MoELayer(n, k, d, 2 * d, 0, T, "bf16", renorm, device="cuda")
    layer.set_capacities(capacity_from_factors([1.0] * n, T, k))
    outs = []
    for full in (False, True):
        if full:
            layer.set_spec_grads(torch.zeros(T * k, d, dtype=torch.bfloat16, device="cuda"),
                                 torch.zeros(T, k, dtype=torch.float32, device="cuda"))
        y, gr = _run(layer, g, dy, 14, y_fill=float("nan"))
        r = layer.routing(T)
        outs.append((gr, r["dl"].clone(), r["dw"].clone()))
    (g1, dl1, dw1), (g2, dl2, dw2) = outs
    assert torch.equal(dl1, dl2) and torch.equal(dw1, dw2)
    for key in g1:
        _bitwise(g2[key], g1[key], key)


@pytest.mark.parametrize("n,k,d,T,alpha", [(64, 1, 1024, 4096, 1.0), (16, 1, 256, 1500, 0.7)])
def test_backward_tail_mode_bitwise(n, k, d, T, alpha, monkeypatch):
    """The backward tail without PDL waits (db1 reduction, drop-only gate-dx pass, gate-weight
    gradient, dA / dX GEMMs overlapping their predecessors; dA in its own buffer) against the
    plain PDL chain (MOE_TAIL=0): every output bitwise equal, over three iterations with
    gradient accumulation and dropped tokens (outputs poisoned first)."""
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    from synth import make_dy, make_layer
    g = {kk: v.cuda() for kk, v in make_layer(n, d, 4 * d, d, T, "bf16").items()}
    dy = make_dy(T, d, "bf16").cuda()
    outs = []
    for tail in ("1", "0"):
        monkeypatch.setenv("MOE_TAIL", tail)
        layer = MoELayer(n, k, d, 4 * d, 0, T, "bf16", 0, device="cuda")
        layer.set_capacities(capacity_from_factors([alpha] * n, T, k))
        grads = None
        for it in range(3):
            y = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
            grads = layer.backward(dy, grads=grads, accumulate=it > 0)
        torch.cuda.synchronize()
        outs.append((y.clone(), {kk: v.clone() for kk, v in grads.items()}))
        layer.close()
    (y1, g1), (y0, g0) = outs
    _bitwise(y1, y0, "y")
    for key in g0:
        _bitwise(g1[key], g0[key], key)


@pytest.mark.gpu
@pytest.mark.parametrize("n,k,d,T,alpha,fusion", [
    (8, 1, 512, 2048, 4.0, 14), (8, 1, 512, 2048, 4.0, 0), (16, 2, 256, 1500, 3.0, 14),
    (16, 2, 256, 1500, 3.0, 0), (8, 1, 256, 2500, 1.0, 15)])
def test_half_tiles_bitwise(n, k, d, T, alpha, fusion, monkeypatch):
    """Remainder m-tiles of <= 128 rows run as M = 128 tiles over the CTA pair
    (MOE_HALF_TILES=1, the default) against full 256-row tiles: every output bitwise equal
    except db1, whose per-CTA row partials split the tile's rows differently (fp32 sums in
    another order, one bf16 rounding: within 1 ulp).  No-drop capacities give remainders of
    every size, so both tile shapes occur in each GEMM."""
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    from synth import make_dy, make_layer
    g = {kk: v.cuda() for kk, v in make_layer(n, d, 4 * d, d, T, "bf16").items()}
    dy = make_dy(T, d, "bf16").cuda()
    outs = []
    for half in ("1", "0"):
        monkeypatch.setenv("MOE_HALF_TILES", half)
        layer = MoELayer(n, k, d, 4 * d, 0, T, "bf16", 0, device="cuda")
        layer.set_capacities(capacity_from_factors([alpha] * n, T, k))
        layer.set_fusion(fusion)
        grads = None
        for it in range(2):
            y = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
            grads = layer.backward(dy, grads=grads, accumulate=it > 0)
        torch.cuda.synchronize()
        outs.append((y.clone(), {kk: v.clone() for kk, v in grads.items()}))
        layer.close()
    (y1, g1), (y0, g0) = outs
    _bitwise(y1, y0, "y")
    for key in g0:
        if key == "db1":
            a, b = g1[key].float(), g0[key].float()
            assert torch.all((a - b).abs() <= b.abs() * 2.0 ** -7 + 1e-30), "db1 beyond 1 ulp"
        else:
            _bitwise(g1[key], g0[key], key)


@pytest.mark.parametrize("n,k,d,f,T,renorm,alpha,fusion", [
    (8, 1, 256, 256, 999, 0, 1.0, 14),      # c5 kind: fused combine, ragged last tile
    (16, 1, 128, 256, 1500, 0, 0.6, 14),    # heavy drops: y rows of dropped tokens zeroed
    (8, 2, 256, 384, 777, 1, 1.0, 14),      # k = 2: two destination rows per x row
    (130, 2, 128, 128, 700, 0, 0.8, 14),    # n > 128 (256-wide gate tile), n % 32 != 0
    (8, 1, 64, 128, 257, 1, 1.25, 0),       # d = 64 (one k-block), no other fusion
    (64, 1, 1024, 512, 4096, 0, 1.0, 14),   # c5 widths, several tiles per CTA
])
def test_cached_dispatch_in_gate_bitwise(n, k, d, f, T, renorm, alpha, fusion):
    """FUSE_CDISP (flag 32): with cached assignments the gate kernel also computes the slots
    and copies the kept x rows into X_buf from its TMA stages.  Every output -- y, all
    gradients, the routing tables, the dispatched X rows and the zeroed pad rows -- is bitwise
    equal to the unfused cached path (dispatch kernel on the side stream); outputs poisoned
    first, two forwards in a row (the second over the first's buffers)."""
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    from synth import make_dy, make_layer
    g = {kk: v.cuda() for kk, v in make_layer(n, d, f, d, T, "bf16").items()}
    dy = make_dy(T, d, "bf16").cuda()
    gen = torch.Generator(device="cpu").manual_seed(11 + n + k)
    cidx = torch.stack([torch.randperm(n, generator=gen)[:k] for _ in range(T)]).int().cuda()
    layer = MoELayer(n, k, d, f, 0, T, "bf16", renorm, device="cuda")
    layer.set_capacities(capacity_from_factors([alpha] * n, T, k))
    layer.set_cached_assignment(cidx)

    def tables():
        r = layer.routing(T)
        rows = r["x_buf"].clone()
        return {kk: r[kk] for kk in ("idx", "fresh_idx", "slot_of", "w", "logits", "kept",
                                     "counts", "token_of_slot")}, rows, r["base"]

    def poison_x():  # every X_buf row NaN: the fused path must write the kept and pad rows
        import ctypes as C
        from paper_2205_01848_b200 import _lib as L
        r = L.Routing()
        L.check(layer.lib.moe_get_routing(layer.h, C.byref(r)), layer.h)
        off = r.x_buf - layer.ws.data_ptr()
        layer.ws[off:off + r.rows * d * 2].view(torch.bfloat16).fill_(float("nan"))

    y0, g0 = _run(layer, g, dy, fusion, y_fill=float("nan"))
    t0, x0, base = tables()
    for it in range(2):
        poison_x()
        y1, g1 = _run(layer, g, dy, fusion | 32, y_fill=float("nan"))
        t1, x1, _ = tables()
        _bitwise(y1, y0, f"y (it {it})")
        for key in g0:
            _bitwise(g1[key], g0[key], f"{key} (it {it})")
        for key in t0:
            assert torch.equal(t1[key], t0[key]), f"{key} (it {it})"
        # X rows of every expert region up to the zeroed pad end (roundup(kept, 64))
        kept = t0["kept"].tolist()
        for e in range(n):
            r1 = base[e] + (kept[e] + 63) // 64 * 64
            _bitwise(x1[base[e]:r1], x0[base[e]:r1], f"X rows of expert {e}")
    assert int(t0["slot_of"].lt(0).sum()) > 0 or alpha >= 1.0


@pytest.mark.parametrize("n,k,d,T,alpha,fusion", [
    (8, 1, 512, 2048, 4.0, 14), (16, 2, 256, 1500, 3.0, 0), (8, 1, 256, 2500, 1.0, 15),
    (64, 1, 1024, 8192, 1.0, 14)])
def test_wgrad_k_tail_trim_bitwise(n, k, d, T, alpha, fusion, monkeypatch):
    """The weight-gradient GEMMs issue only the 16-deep MMAs of their last token k-block that
    hold kept tokens (default) against all four (MOE_NO_KTRIM=1): the skipped MMAs would add
    products of zero pad rows, so every output is bitwise equal -- kept counts of every
    residue mod 64 occur (no-drop capacities), with gradient accumulation on the second
    iteration and the gather fusion (flag 1) in one case."""
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    from synth import make_dy, make_layer
    g = {kk: v.cuda() for kk, v in make_layer(n, d, 4 * d, d, T, "bf16").items()}
    dy = make_dy(T, d, "bf16").cuda()
    outs = []
    for trim in ("0", "1"):
        monkeypatch.setenv("MOE_NO_KTRIM", trim)
        layer = MoELayer(n, k, d, 4 * d, 0, T, "bf16", 0, device="cuda")
        layer.set_capacities(capacity_from_factors([alpha] * n, T, k))
        layer.set_fusion(fusion)
        grads = None
        for it in range(2):
            y = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
            grads = layer.backward(dy, grads=grads, accumulate=it > 0)
        torch.cuda.synchronize()
        kept = layer.routing(T)["kept"]
        outs.append((y.clone(), {kk: v.clone() for kk, v in grads.items()}))
        layer.close()
    assert bool(((kept % 16) != 0).any())
    (y1, g1), (y0, g0) = outs
    _bitwise(y1, y0, "y")
    for key in g0:
        _bitwise(g1[key], g0[key], key)
