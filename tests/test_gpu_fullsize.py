"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (default
fusion flags, uniform synthetic inputs of the bench).

* c3 (the bench workload) and c5 (c3 in cached mode): the WHOLE layer against the complete
  fp64 oracle on the complete batch -- routing bit-exact (decisions from the kernel's fp32
  logits), and y, dx, dW_g, every expert's dW1 / db1 / dW2 / db2 (also normalised per
  expert), dl and dw (also per token) within the bf16 budget.  The oracle's fp64 run takes
  ~15 GB of host memory and a few tens of seconds on the box's 16 cores.
* c4 (262,144 tokens, top-2, d 2048, f 8192): the complete oracle would need ~70 GB of fp64
  gradient buffers and ~106 TFLOP, so it runs on sub-problems whose outputs provably equal
  the full problem's on the rows compared (renormalised weights depend only on a token's own
  selected logits, a token's outputs depend on the batch only through which of its pairs
  were kept, an expert's gradients only on its kept rows): sampled tokens' logits / w / y /
  dw / dl / dx, and the complete dW1 / db1 / dW2 / db2 of two experts (one at capacity with
  drops), with the whole batch's routing bit-exact.

ReLU' decisions are the oracle's own except inside the fp32 rounding band of an element
(checked_relu_mask: any disagreement outside it fails)."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from parity_util import (TOL, checked_relu_mask, kernel_relu_mask, rel, rel_rows, rel_scaled,
                         token_scales)
from synth import get_config, make_dy, make_layer, perturb_cached, to_numpy64

pytestmark = pytest.mark.gpu

N_SAMPLES = 24


def _setup(name):
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    cfg = get_config(name)
    n, k, d, f, do, T = cfg.n_experts, cfg.top_k, cfg.d_model, cfg.d_ff, cfg.d_out, cfg.tokens
    g = make_layer(n, d, f, do, T, cfg.dtype, "uniform", device="cuda")
    layer = MoELayer(n, k, d, f, do, T, cfg.dtype, cfg.renormalize, device="cuda")
    caps = capacity_from_factors([cfg.alpha] * n, T, k)
    layer.set_capacities(caps)
    return cfg, g, layer, caps


def _check_routing(cfg, rt, caps, cidx=None):
    """Whole batch: fresh idx = top-k of the kernel's logits (reading 3, decision in the
    kernel's precision), slot_of = the oracle's token-major grouping (reading 6), kept."""
    n, k = cfg.n_experts, cfg.top_k
    lg = rt["logits"].cpu().double().numpy()
    fresh = O.topk_sorted(lg, k)
    assert np.array_equal(rt["fresh_idx"].cpu().numpy(), fresh)
    idx = fresh if cidx is None else cidx
    assert np.array_equal(rt["idx"].cpu().numpy(), idx)
    ort = O.route(idx, caps, n)
    assert np.array_equal(rt["slot_of"].cpu().numpy(), ort.slot_of)
    assert np.array_equal(rt["kept"].cpu().numpy().astype(np.int64), ort.kept)
    assert np.array_equal(rt["counts"].cpu().numpy().astype(np.int64), ort.counts)
    return lg, idx, ort


def _full_layer_vs_oracle(name, cached_frac=None):
    cfg, g, layer, caps = _setup(name)
    n, k, T = cfg.n_experts, cfg.top_k, cfg.tokens
    dy = make_dy(T, cfg.d_out, cfg.dtype, device="cuda")
    x64 = to_numpy64(g["x"])
    p64 = {kk: to_numpy64(v) for kk, v in g.items() if kk != "x"}
    cidx = None
    if cached_frac is not None:   # the cached table is an input: the oracle's top-k, perturbed
        fresh0 = O.topk_sorted(O.gate_logits(x64, p64["w_gate"]), k)
        cidx = np.ascontiguousarray(perturb_cached(fresh0, n, cached_frac), dtype=np.int32)
        layer.set_cached_assignment(torch.from_numpy(cidx).cuda())
    y = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    rt = layer.routing(T)
    stats = layer.stats()
    grads = layer.backward(dy)
    torch.cuda.synchronize()
    assert layer.check_flags()[1] == 0
    rb = layer.routing(T)        # dl / dw of the backward
    lg, idx, ort = _check_routing(cfg, rt, caps, cidx)
    assert int(ort.drops) > 0 and stats["drops"] == int(ort.drops)
    st = O.moe_forward(x64, p64, k, caps, cfg.renormalize, logits=lg, cached_idx=cidx,
                       emulate_bf16=(cfg.dtype == "bf16"))
    assert stats["hit_count"] == st.hit_count
    if cidx is not None:
        assert 0 < st.hit_count < T
    mask = checked_relu_mask(st, kernel_relu_mask(rt, st), name)
    del rt
    gr = O.moe_backward(st, to_numpy64(dy), relu_mask=mask)
    tol = TOL[cfg.dtype]
    errs = {"logits": rel(lg, O.gate_logits(x64, p64["w_gate"])), "w": rel(rb["w"].cpu().numpy(), st.w),
            "y": rel(to_numpy64(y), st.y)}
    for key in ("dx", "dw_gate", "dw1", "db1", "dw2", "db2"):
        errs[key] = rel(to_numpy64(grads[key]), gr[key])
    for key in ("dw1", "db1", "dw2", "db2"):
        errs[key + "/expert"] = rel_rows(to_numpy64(grads[key]), gr[key])
    s_dw, s_dl = token_scales(st, to_numpy64(dy))
    for key, sc in (("dl", s_dl), ("dw", s_dw)):
        v = rb[key].cpu().double().numpy()
        errs[key] = rel(v, gr[key])
        errs[key + "/elem"] = rel_scaled(v, gr[key], sc)
    lim = {kk: (1e-5 if kk in ("logits", "w") else tol) for kk in errs}
    bad = {kk: v for kk, v in errs.items() if not v <= lim[kk]}
    assert not bad, f"{name} full-size parity failures {bad} (all: {errs})"
    return errs


@pytest.mark.timeout(900)
def test_c3_full_size_whole_layer_vs_oracle():
    """c3 (the bench workload: 64 experts, top-1, d 1024, f 4096, 65,536 tokens, bf16, raw
    softmax weights so the gate trains): every output and gradient of the layer against the
    complete fp64 oracle."""
    errs = _full_layer_vs_oracle("c3")
    print("c3 full-size errors", errs)


@pytest.mark.timeout(900)
def test_c5_full_size_cached_whole_layer_vs_oracle():
    """c5 (c3 with sample-assignment caching) in the bench's launch configuration,
    3 % of the cached rows stale: dispatch follows the cached indices, fresh top-k and hit
    count the kernel's logits, and every output and gradient matches the complete oracle."""
    errs = _full_layer_vs_oracle("c5", cached_frac=0.03)
    print("c5 full-size errors", errs)


# ----------------------------------------------------------------------------------------
# c4: sub-problems of the oracle (renormalised weights, see module docstring)
# ----------------------------------------------------------------------------------------
def _sub_oracle(cfg, g, toks, lg, idx, slot_of, keep=None, dy=None, rt_h=None, base=None):
    """The oracle on tokens `toks` (ascending) over the experts they use, renumbered 0..m-1.
    keep: if given, only pairs whose expert is in `keep` are real experts; every other pair
    goes to one extra zero-weight expert with capacity 0 (dropped), whose per-token logit
    column is that pair's real logit -- so renormalised w, the kept rows, dO = w dy and the
    kept experts' gradients are exactly the full problem's (dl / dx of such a run are not).
    Capacities keep exactly the pairs the full problem kept (a prefix of each expert's
    tokens in token order).  Returns (state, grads or None, expert renumbering)."""
    assert cfg.renormalize == 1, "sub-problems need renormalised weights (reading 4)"
    n, k = cfg.n_experts, cfg.top_k
    toks = sorted(int(t) for t in toks)
    used = sorted({int(idx[t, r]) for t in toks for r in range(k)}) if keep is None else \
        sorted(int(e) for e in keep)
    j_of = {e: j for j, e in enumerate(used)}
    m = len(used) + (1 if keep is not None else 0)
    dummy = len(used)
    sub_idx = np.zeros((len(toks), k), np.int32)
    sub_l = np.full((len(toks), m), -1e30)
    caps = [0] * m
    for i, t in enumerate(toks):
        outside = 0
        for r in range(k):
            e = int(idx[t, r])
            if e in j_of:
                j = j_of[e]
                if slot_of[t, r] >= 0:
                    caps[j] += 1
            else:
                j = dummy
                outside += 1
                assert outside <= 1, "one dummy expert holds at most one pair per token"
            sub_idx[i, r] = j
            sub_l[i, j] = lg[t, e]
    d, f, do = cfg.d_model, cfg.d_ff, cfg.d_out
    params = {"w_gate": np.zeros((m, d)), "w1": np.zeros((m, f, d)), "b1": np.zeros((m, f)),
              "w2": np.zeros((m, do, f)), "b2": np.zeros((m, do))}
    for e, j in j_of.items():
        params["w_gate"][j] = to_numpy64(g["w_gate"][e])
        for key in ("w1", "b1", "w2", "b2"):
            params[key][j] = to_numpy64(g[key][e])
    st = O.moe_forward(to_numpy64(g["x"][toks]), params, k, caps, 1, logits=sub_l,
                       cached_idx=sub_idx, emulate_bf16=(cfg.dtype == "bf16"))
    gr = None
    if dy is not None:   # kernel ReLU' rows in the oracle's slot order (token order)
        rows = [[] for _ in range(m)]
        for i, t in enumerate(toks):
            for r in range(k):
                if st.routing.slot_of[i, r] >= 0:
                    e = int(idx[t, r])
                    rows[sub_idx[i, r]].append(
                        rt_h[base[e] + int(slot_of[t, r])].float().cpu().numpy() > 0)
        kmask = [np.array(rw, bool).reshape(len(rw), f) for rw in rows]
        mask = checked_relu_mask(st, kmask, "c4 sub-problem")
        gr = O.moe_backward(st, to_numpy64(dy[toks]), relu_mask=mask)
    return st, gr, j_of


def _samples(ort, T, k, n_samples=N_SAMPLES):
    rng = np.random.default_rng(1848)
    kept_all = np.where((ort.slot_of >= 0).all(axis=1))[0]
    some_drop = np.where((ort.slot_of < 0).any(axis=1))[0]
    pick = list(rng.choice(kept_all, n_samples - 6, replace=False))
    if len(some_drop):
        pick += list(rng.choice(some_drop, min(6, len(some_drop)), replace=False))
    return sorted(int(t) for t in pick)


@pytest.mark.timeout(1200)
def test_c4_full_size_vs_oracle():
    """c4 (128 experts, top-2, d 2048, f 8192, 262,144 tokens, bf16) on one GPU: routing
    bit-exact over the whole batch; sampled tokens (all-kept, partly and fully dropped) --
    logits, w, y, dw, dl, dx -- and two experts' complete weight and bias gradients (the most
    loaded expert, at capacity with drops, and the least loaded) against the oracle."""
    cfg, g, layer, caps = _setup("c4")
    n, k, T = cfg.n_experts, cfg.top_k, cfg.tokens
    dy = make_dy(T, cfg.d_out, cfg.dtype, device="cuda")
    y = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    rt = layer.routing(T)
    grads = layer.backward(dy)
    torch.cuda.synchronize()
    assert layer.check_flags()[1] == 0
    rb = layer.routing(T)
    lg, idx, ort = _check_routing(cfg, rt, caps)
    h_buf, base = rt["h_buf"], rt["base"]
    w = rt["w"].cpu().double().numpy()
    dl = rb["dl"].cpu().double().numpy()
    dw = rb["dw"].cpu().double().numpy()
    wg = to_numpy64(g["w_gate"])
    tol = TOL[cfg.dtype]
    errs = {}
    # sampled tokens, one oracle sub-problem per token (its own experts)
    for t in _samples(ort, T, k):
        st, gr, j_of = _sub_oracle(cfg, g, [t], lg, idx, ort.slot_of, dy=dy, rt_h=h_buf,
                                   base=base)
        assert np.array_equal(st.routing.slot_of[0] >= 0, ort.slot_of[t] >= 0)
        cols = [j_of[int(e)] for e in idx[t]]
        s_dw, s_dl = token_scales(st, to_numpy64(dy[t:t + 1]))
        e_ = {"dw/elem": rel_scaled(dw[t], gr["dw"][0], s_dw[0]),
              "dl/elem": rel_scaled(dl[t][idx[t]], gr["dl"][0][cols], s_dl[0][cols]),
              "logits": rel(lg[t], O.gate_logits(to_numpy64(g["x"][t:t + 1]), wg)[0]),
              "w": rel(w[t], st.w[0]), "y": rel(to_numpy64(y[t]), st.y[0]),
              "dx": rel(to_numpy64(grads["dx"][t]), gr["dx"][0])}
        # renormalised: dl is exactly zero off the selected experts (reading 4)
        off = np.ones(n, bool)
        off[idx[t]] = False
        assert (dl[t][off] == 0).all(), t
        for kk, v in e_.items():
            errs[kk] = max(errs.get(kk, 0.0), v)
    kept = rt["kept"].cpu().numpy()
    counts = rt["counts"].cpu().numpy()
    e_hi = int(np.argmax(counts))
    e_lo = int(np.argmin(counts))
    assert counts[e_hi] > caps[e_hi] and kept[e_hi] == caps[e_hi]   # at capacity, drops
    for e in (e_hi, e_lo):
        toks = np.where(((idx == e) & (ort.slot_of >= 0)).any(axis=1))[0]
        assert len(toks) == kept[e]
        st, gr, j_of = _sub_oracle(cfg, g, toks, lg, idx, ort.slot_of, keep=[e], dy=dy,
                                   rt_h=h_buf, base=base)
        j = j_of[e]
        assert int(st.routing.kept[j]) == kept[e]
        for key in ("dw1", "db1", "dw2", "db2"):
            errs[f"{key}[{e}]"] = rel(to_numpy64(grads[key][e]), gr[key][j])
    lim = {kk: (1e-5 if kk in ("logits", "w") else tol) for kk in errs}
    bad = {kk: v for kk, v in errs.items() if not v <= lim[kk]}
    assert not bad, f"c4 parity failures {bad} (all: {errs})"
    print("c4 errors", errs)


@pytest.mark.timeout(600, method="thread")
@pytest.mark.parametrize("R,transport", [(2, "peer"), (4, "peer"), (2, "nccl")])
def test_c3_per_rank_expert_parallel_bitwise(R, transport):
    """The bench's N > 1 configuration at its per-rank size (c3 per rank: 65,536 tokens per
    rank, n / R experts per rank; peer transport with return rows and the fused dispatch
    backward, or the NCCL-style transport bench.py falls back to), as R virtual ranks on one
    GPU: routing, y, dx and each owner's expert gradients bitwise equal to the single-GPU
    layer on the concatenated batch."""
    from test_gpu_ep import _check_virtual, _run_virtual
    cfg = get_config("c3")
    out, ref = _run_virtual(R, cfg.n_experts, cfg.top_k, cfg.tokens, cfg.d_model, cfg.d_ff,
                            cfg.dtype, cfg.renormalize, transport=transport, fusion=6)
    _check_virtual(out, ref, R, cfg.n_experts, cfg.dtype)
