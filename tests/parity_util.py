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


def rel_rows(a, b, floor=1e-3):
    """Row-wise (first axis) error: max over rows of ||a_i-b_i||_inf / ||b_i||_inf, each row
    normalised by its own magnitude (per expert for the [n, ...] gradient tensors, per token
    for dl / dw).  Rows whose own magnitude is below `floor` x the tensor's are normalised by
    floor x the tensor's magnitude instead (so exact-zero rows must stay ~zero)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    a2 = a.reshape(a.shape[0], -1)
    b2 = b.reshape(b.shape[0], -1)
    glob = np.abs(b2).max()
    if glob == 0:
        return float(np.abs(a2).max())
    den = np.maximum(np.abs(b2).max(axis=1), floor * glob)
    return float((np.abs(a2 - b2).max(axis=1) / den).max())


def token_scales(st, dy, lam_g=None):
    """Per-element condition scales of dw [T,k] and dl [T,n] (DESIGN.md §2 "error metric"):
    dw[t,r] = <dy[t], O[row]> is a d_out-term dot product, so an input perturbation of
    relative size eps moves it by at most eps * sum_i |dy_i||O_i| = s_dw[t,r] (that, not |dw|,
    is its natural scale: |dw| can be ~0 by cancellation).  dl is a fixed combination of the
    dw's: renorm dl_{i_r} = w_r (dw_r - sum_s w_s dw_s) -> w_r (s_dw_r + sum_s w_s s_dw_s);
    raw dl_j = p_j (dp_j - sum_s w_s dw_s) -> p_j (s_dp_j + sum_s w_s s_dw_s); with the Eq. 3
    balance term (g = lam_g [n]) p_j (|g_j| + sum_i p_i |g_i|) is added."""
    dy = np.asarray(dy, np.float64)
    T, k, n = st.x.shape[0], st.k, st.n
    s_dw = np.zeros((T, k))
    for e in range(n):
        Oe = np.abs(st.O[e])
        for j, code in enumerate(st.routing.token_of_slot[e]):
            t, r = divmod(int(code), k)
            t -= st.token_offset
            s_dw[t, r] = float(np.abs(dy[t]) @ Oe[j])
    w, idx = st.w, st.idx
    c = (w * s_dw).sum(axis=1)
    s_dl = np.zeros((T, n))
    rows = np.arange(T)
    if st.renormalize:
        for r in range(k):
            s_dl[rows, idx[:, r]] += w[:, r] * (s_dw[:, r] + c)
    else:
        sdp = np.zeros((T, n))
        for r in range(k):
            sdp[rows, idx[:, r]] += s_dw[:, r]
        s_dl = st.p * (sdp + c[:, None])
    if lam_g is not None:
        ag = np.abs(np.asarray(lam_g, np.float64))
        s_dl += st.p * (ag[None, :] + (st.p * ag[None, :]).sum(axis=1, keepdims=True))
    return s_dw, s_dl


def rel_scaled(a, b, scale):
    """max |a - b| / scale elementwise; where scale is 0 the values must agree exactly."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    err = np.abs(a - b)
    z = scale <= 0
    if (err[z] > 0).any():
        return float("inf")
    return float((err[~z] / scale[~z]).max()) if (~z).any() else 0.0


# ReLU' decisions (DESIGN.md §2 "ReLU' decisions in parity").  The kernel accumulates
# A = X W1^T + b1 in fp32 from exact bf16/fp32 products; its rounding error on one element is
# far below RELU_BOUND_C * u32 * (sum_j |x_j||w_j| + |b|) (the random-walk estimate of fp32
# summation error over d terms is ~ u32 * d / (32*sqrt(6)) for these inputs, the bound is
# >= 10x that).  Only elements whose fp64 A lies inside that band may take the kernel's
# sign; a disagreement outside it is a kernel bug and fails the test.
U32 = 2.0 ** -24
RELU_BOUND_C = 8.0
RELU_FLIP_FRAC = 1e-6


def checked_relu_mask(st, kernel_mask, what=""):
    """The ReLU' mask the oracle's backward should use: the oracle's own A > 0, except on
    elements where the kernel's decision (its stored H > 0) differs AND the oracle's |A| is
    inside the fp32 rounding band of that element -- those take the kernel's decision, like
    routing takes the kernel's fp32 logits.  Asserts every disagreement is inside the band and
    that they are rare (<= max(3, RELU_FLIP_FRAC * elements))."""
    out = []
    flips = total = 0
    for e in range(st.n):
        A = st.A[e]
        km = np.asarray(kernel_mask[e], bool).reshape(A.shape)
        dis = km != (A > 0)
        total += A.size
        if dis.any():
            kept = A.shape[0]
            X = st.X[e][:kept]
            W1 = np.asarray(st.params["w1"][e], np.float64)
            b1 = np.asarray(st.params["b1"][e], np.float64)
            rr, cc = np.nonzero(dis)
            band = RELU_BOUND_C * U32 * ((np.abs(X[rr]) * np.abs(W1[cc])).sum(axis=1)
                                         + np.abs(b1[cc]))
            a = np.abs(A[rr, cc])
            assert (a <= band).all(), (
                f"{what} expert {e}: kernel ReLU' decision differs from the oracle outside the "
                f"fp32 rounding band: |A| {a[a > band][:5]} > band {band[a > band][:5]} at "
                f"(row, col) {list(zip(rr[a > band][:5], cc[a > band][:5]))}")
            flips += int(dis.sum())
        out.append(km)
    assert flips <= max(3, RELU_FLIP_FRAC * total), f"{what}: {flips} ReLU' flips of {total}"
    return out


def kernel_relu_mask(rt, st):
    """The kernel's ReLU' decisions (stored H > 0) in the oracle's per-expert slot order."""
    n = st.n
    return [(rt["h_buf"][rt["base"][e]: rt["base"][e] + int(st.routing.kept[e])].float() > 0)
            .cpu().numpy() for e in range(n)]


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
    # ReLU' decisions: the oracle's own, except inside the fp32 rounding band (checked)
    mask = None
    if len(rt_f["base"]) == n + 1:
        mask = checked_relu_mask(st, kernel_relu_mask(rt_f, st), "run_pair")
    gr = O.moe_backward(st, to_numpy64(dy), relu_mask=mask)
    gpu["scales"] = token_scales(st, to_numpy64(dy))
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
    # weak entries: expert gradients normalised per expert (lightly loaded experts), dl / dw
    # per token (confident routers)
    for key in ("dw1", "db1", "dw2", "db2"):
        if key in gpu:
            errs[key + "/expert"] = rel_rows(gpu[key], gr[key])
    if "scales" in gpu:
        s_dw, s_dl = gpu["scales"]
        errs["dl/elem"] = rel_scaled(gpu["routing"]["dl"], gr["dl"], s_dl)
        errs["dw/elem"] = rel_scaled(gpu["routing"]["dw"], gr["dw"], s_dw)
    # logits and gate weights are fp32 in both dtypes
    lim = {kk: (1e-5 if kk in ("logits", "w") else tol) for kk in errs}
    bad = {kk: v for kk, v in errs.items() if kk not in skip and not v <= lim[kk]}
    assert not bad, f"parity failures {bad} (all: {errs})"
    return errs
