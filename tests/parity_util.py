"""Shared helpers of the GPU-vs-oracle parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import moe_oracle as O
from synth import make_dy, make_layer, to_numpy64

TOL = {"f32": 1e-5, "bf16": 2e-2}


def _np(v):
    if not torch.is_tensor(v):
        return v
    if v.dtype == torch.bfloat16:
        v = v.float()
    return v.cpu().numpy()


def rel(a, b):
    """Per-tensor ||a-b||_inf / ||b||_inf (reading 13)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    den = np.abs(b).max()
    num = np.abs(a - b).max()
    if den == 0:
        return float(num)
    return float(num / den)


def run_pair(n, k, d, f, T, dtype, caps, renorm=1, regime="uniform", d_out=None,
             cached=None, dev="cuda", layer=None, max_tokens=None, seed_offset=0):
    """Run the CUDA layer and the oracle on the same seeded inputs.
    cached: None, or a callable(fresh_idx_oracle) -> cached idx array [T,k]."""
    from paper_2205_01848_b200 import MoELayer
    do = d_out or d
    cpu = make_layer(n, d, f, do, T, dtype, regime, seed_offset=seed_offset)
    dy = make_dy(T, do, dtype, seed_offset=seed_offset)
    if layer is None:
        layer = MoELayer(n, k, d, f, d_out or 0, max_tokens or max(T, 1), dtype, renorm, device=dev)
    layer.set_capacities(caps)
    g = {kk: v.to(dev) for kk, v in cpu.items()}
    x64 = to_numpy64(cpu["x"])
    p64 = {kk: to_numpy64(v) for kk, v in cpu.items() if kk != "x"}
    cidx = None
    if cached is not None:
        l_ref = O.gate_logits(x64, p64["w_gate"])
        cidx = np.ascontiguousarray(cached(O.topk_sorted(l_ref, k)), dtype=np.int32)
        layer.set_cached_assignment(torch.from_numpy(cidx).to(dev))
    else:
        layer.set_cached_assignment(None)
    y = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    rt_f = layer.routing(T)
    st_flags = layer.check_flags()
    stats = layer.stats()
    grads = layer.backward(dy.to(dev))
    torch.cuda.synchronize()
    rt = layer.routing(T)
    gpu = dict(y=to_numpy64(y), **{kk: to_numpy64(v) for kk, v in grads.items()})
    gpu["routing"] = {kk: _np(v) for kk, v in rt.items()}
    gpu["routing_fwd"] = {kk: _np(v) for kk, v in rt_f.items()}
    gpu["stats"] = stats
    gpu["flags"] = st_flags
    # oracle: routing decisions from the GPU's fp32 logits (north star), fp64 values
    gl = gpu["routing_fwd"]["logits"].astype(np.float64)
    st = O.moe_forward(x64, p64, k, caps, renorm, cached_idx=cidx, logits=gl,
                       emulate_bf16=(dtype == "bf16"))
    # the ReLU' decision in the kernel's precision (its stored H > 0), like routing from its
    # fp32 logits: both sides take every integer decision alike
    rf = gpu["routing_fwd"]
    mask = None
    if len(rf["base"]) == n + 1 and "h_buf" in rf:
        mask = [rf["h_buf"][rf["base"][e]: rf["base"][e] + int(st.routing.kept[e])] > 0
                for e in range(n)]
    gr = O.moe_backward(st, to_numpy64(dy), relu_mask=mask)
    own_logits = O.gate_logits(x64, p64["w_gate"])
    return layer, gpu, st, gr, own_logits


def assert_routing_exact(gpu, st, k, check_token_of_slot=True):
    r = gpu["routing_fwd"]
    assert np.array_equal(r["fresh_idx"], st.fresh_idx), "fresh top-k differs"
    assert np.array_equal(r["idx"], st.idx), "dispatch idx differs"
    assert np.array_equal(r["slot_of"], st.routing.slot_of), "slot_of differs"
    assert np.array_equal(r["counts"].astype(np.int64), st.routing.counts), "counts differ"
    assert np.array_equal(r["kept"].astype(np.int64), st.routing.kept), "kept differs"
    assert gpu["stats"]["drops"] == st.routing.drops
    assert gpu["stats"]["hit_count"] == st.hit_count
    if not check_token_of_slot:   # EP: token_of_slot indexes the send layout
        return
    base = r["base"]
    tos = r["token_of_slot"]
    for e in range(len(st.routing.token_of_slot)):
        exp = np.array(st.routing.token_of_slot[e], np.int64)
        got = tos[base[e]: base[e] + len(exp)].astype(np.int64)
        assert np.array_equal(got, exp), f"token_of_slot differs for expert {e}"


def assert_values(gpu, st, gr, own_logits, dtype, skip=()):
    tol = TOL[dtype]
    r = gpu["routing_fwd"]
    errs = {
        "logits": rel(r["logits"], own_logits),
        "w": rel(r["w"], st.w),
        "y": rel(gpu["y"], st.y),
        "dw": rel(gpu["routing"]["dw"], gr["dw"]),
        "dl": rel(gpu["routing"]["dl"], gr["dl"]),
    }
    for key in ("dx", "dw_gate", "dw1", "db1", "dw2", "db2"):
        if key in gpu:
            errs[key] = rel(gpu[key], gr[key])
    # logits and gate weights are fp32 in both dtypes
    lim = {kk: (1e-5 if kk in ("logits", "w") else tol) for kk in errs}
    bad = {kk: v for kk, v in errs.items() if kk not in skip and not v <= lim[kk]}
    assert not bad, f"parity failures {bad} (all: {errs})"
    return errs
