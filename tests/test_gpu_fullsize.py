"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (default
fusion flags, uniform synthetic inputs of the bench): the whole routing checked bit-exact
against the oracle (top-k of the kernel's fp32 logits, token-major capacity grouping over the
complete batch), and sampled tokens' logits / gate weights / y (and, at c3, dw, dl, dx) against
the oracle run on those tokens alone.

A token's outputs depend on the rest of the batch only through which of its pairs were kept,
so sampled tokens go to the oracle as small batches whose capacities keep exactly their kept
pairs (all-kept tokens together, all-dropped tokens together, mixed tokens one at a time);
only the experts they use are widened to fp64 (the full weights would not fit in fp64 host
memory at c4)."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from parity_util import TOL, rel
from synth import get_config, make_dy, make_layer, to_numpy64

pytestmark = pytest.mark.gpu

N_SAMPLES = 24


class _Experts:
    """Per-expert fp64 copies of a device weight tensor [n, ...], fetched only for the
    experts in `used`; every other expert is a zero-stride array of the right shape (it
    multiplies zero rows).  np.asarray() sees a zero-copy broadcast of the full shape (the
    oracle reads its .shape, and allocates its gradient buffers from it at c3)."""

    def __init__(self, t, used):
        self.t, self.used, self.cache = t, set(int(e) for e in used), {}
        self.shape = tuple(t.shape)
        self.dummy = np.broadcast_to(np.zeros(1), self.shape[1:])

    def __getitem__(self, e):
        e = int(e)
        if e not in self.used:
            return self.dummy
        if e not in self.cache:
            self.cache[e] = to_numpy64(self.t[e])
        return self.cache[e]

    def __array__(self, dtype=None, copy=None):
        return np.broadcast_to(np.zeros(1, dtype or np.float64), self.shape)


def _setup(name):
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    cfg = get_config(name)
    n, k, d, f, do, T = cfg.n_experts, cfg.top_k, cfg.d_model, cfg.d_ff, cfg.d_out, cfg.tokens
    g = make_layer(n, d, f, do, T, cfg.dtype, "uniform", device="cuda")
    layer = MoELayer(n, k, d, f, do, T, cfg.dtype, cfg.renormalize, device="cuda")
    caps = capacity_from_factors([cfg.alpha] * n, T, k)
    layer.set_capacities(caps)
    return cfg, g, layer, caps


def _check_routing(cfg, rt, caps):
    """Whole batch: idx = top-k of the kernel's logits (reading 3, decision in the kernel's
    precision), slot_of = the oracle's token-major grouping (reading 6), kept counts."""
    n, k = cfg.n_experts, cfg.top_k
    lg = rt["logits"].cpu().double().numpy()
    idx = O.topk_sorted(lg, k)
    assert np.array_equal(rt["idx"].cpu().numpy(), idx)
    ort = O.route(idx, caps, n)
    assert np.array_equal(rt["slot_of"].cpu().numpy(), ort.slot_of)
    assert np.array_equal(rt["kept"].cpu().numpy().astype(np.int64), ort.kept)
    return lg, idx, ort


def _group_oracle(cfg, g, toks, lg, idx, slot_of, h_rows=None, dy=None, cached=False):
    """The oracle on the tokens `toks` alone (ascending), with capacities that keep exactly
    their kept pairs: callers pass groups in which every pair is kept, or every pair
    dropped, or a single token."""
    n, k = cfg.n_experts, cfg.top_k
    caps = [0] * n
    for t in toks:
        for r in range(k):
            if slot_of[t, r] >= 0:
                caps[int(idx[t, r])] += 1
    used = [e for e in range(n) if caps[e]]
    params = {"w_gate": to_numpy64(g["w_gate"])}
    for key in ("w1", "b1", "w2", "b2"):
        params[key] = _Experts(g[key], used)
    st = O.moe_forward(to_numpy64(g["x"][toks]), params, k, caps, cfg.renormalize,
                       logits=lg[toks], emulate_bf16=(cfg.dtype == "bf16"),
                       cached_idx=np.ascontiguousarray(idx[toks]) if cached else None)
    gr = None
    if dy is not None:   # ReLU' decisions from the kernel's H rows, in the oracle's slot order
        rows = [[] for _ in range(n)]
        for j, t in enumerate(toks):
            for r in range(k):
                if st.routing.slot_of[j, r] >= 0:
                    rows[int(idx[t, r])].append(h_rows[(t, r)] > 0)
        mask = [np.array(rw, bool).reshape(len(rw), cfg.d_ff) for rw in rows]
        gr = O.moe_backward(st, to_numpy64(dy[toks]), relu_mask=mask)
    return st, gr


def _samples(ort, T, k):
    rng = np.random.default_rng(1848)
    kept_all = np.where((ort.slot_of >= 0).all(axis=1))[0]
    some_drop = np.where((ort.slot_of < 0).any(axis=1))[0]
    pick = list(rng.choice(kept_all, N_SAMPLES - 4, replace=False))
    if len(some_drop):
        pick += list(rng.choice(some_drop, min(4, len(some_drop)), replace=False))
    return sorted(int(t) for t in pick)


@pytest.mark.timeout(600)
def test_c3_full_size_forward_backward_vs_oracle():
    """c3 (the bench workload: 64 experts, top-1, d 1024, f 4096, 65,536 tokens, bf16)."""
    cfg, g, layer, caps = _setup("c3")
    n, k, T = cfg.n_experts, cfg.top_k, cfg.tokens
    dy = make_dy(T, cfg.d_out, cfg.dtype, device="cuda")
    y = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    rt = layer.routing(T)
    h_buf, base = rt["h_buf"], rt["base"]
    grads = layer.backward(dy)
    torch.cuda.synchronize()
    assert layer.check_flags()[1] == 0
    lg, idx, ort = _check_routing(cfg, rt, caps)
    rb = layer.routing(T)        # dl / dw of the backward
    dl, dw = rb["dl"].cpu().double().numpy(), rb["dw"].cpu().double().numpy()
    w = rt["w"].cpu().double().numpy()
    wg = to_numpy64(g["w_gate"])
    tol = TOL[cfg.dtype]
    samples = _samples(ort, T, k)
    h_rows = {(t, r): h_buf[base[int(idx[t, r])] + int(ort.slot_of[t, r])].float().cpu().numpy()
              for t in samples for r in range(k) if ort.slot_of[t, r] >= 0}
    kept = [t for t in samples if (ort.slot_of[t] >= 0).all()]
    dropped = [t for t in samples if (ort.slot_of[t] < 0).all()]
    assert kept and dropped and len(kept) + len(dropped) == len(samples)   # k = 1
    for grp in (kept, dropped):
        st, gr = _group_oracle(cfg, g, grp, lg, idx, ort.slot_of, h_rows, dy)
        assert np.array_equal(st.routing.slot_of >= 0, ort.slot_of[grp] >= 0)
        for j, t in enumerate(grp):
            assert rel(lg[t], O.gate_logits(to_numpy64(g["x"][t:t + 1]), wg)[0]) <= 1e-5, t
            assert rel(w[t], st.w[j]) <= 1e-5, t
            assert rel(to_numpy64(y[t]), st.y[j]) <= tol, t
            assert rel(dw[t], gr["dw"][j]) <= tol, t     # <dy, O> over bf16-stored O
            assert rel(dl[t], gr["dl"][j]) <= tol, t
            assert rel(to_numpy64(grads["dx"][t]), gr["dx"][j]) <= tol, t


@pytest.mark.timeout(900)
def test_c4_full_size_forward_vs_oracle():
    """c4 (128 experts, top-2, d 2048, f 8192, 262,144 tokens, bf16) on one GPU: routing
    bit-exact over the whole batch, sampled tokens' logits / w / y against the oracle, and
    the backward runs clean (device flags) at this size."""
    cfg, g, layer, caps = _setup("c4")
    n, k, T = cfg.n_experts, cfg.top_k, cfg.tokens
    y = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    rt = layer.routing(T)
    torch.cuda.synchronize()
    lg, idx, ort = _check_routing(cfg, rt, caps)
    w = rt["w"].cpu().double().numpy()
    wg = to_numpy64(g["w_gate"])
    for t in _samples(ort, T, k):   # one token per oracle call (mixed kept / dropped pairs)
        st, _ = _group_oracle(cfg, g, [t], lg, idx, ort.slot_of)
        assert np.array_equal(st.routing.slot_of[0] >= 0, ort.slot_of[t] >= 0)
        assert rel(lg[t], O.gate_logits(to_numpy64(g["x"][t:t + 1]), wg)[0]) <= 1e-5, t
        assert rel(w[t], st.w[0]) <= 1e-5, t
        assert rel(to_numpy64(y[t]), st.y[0]) <= TOL[cfg.dtype], t
    del rt
    grads = layer.backward(make_dy(T, cfg.d_out, cfg.dtype, device="cuda"))
    torch.cuda.synchronize()
    assert layer.check_flags()[1] == 0
    assert all(bool(torch.isfinite(v.float()).all()) for v in grads.values())


@pytest.mark.timeout(600)
def test_c5_full_size_cached_vs_oracle():
    """c5 (c3 shape with sample-assignment caching, §4.2) in the bench's launch
    configuration, with 3 % of the cached rows stale: dispatch follows the cached indices,
    the fresh top-k and the hit count follow the kernel's logits, the whole batch's grouping
    is the oracle's, and sampled tokens' y and dx match the oracle in cached mode."""
    from synth import perturb_cached
    cfg, g, layer, caps = _setup("c5")
    n, k, T = cfg.n_experts, cfg.top_k, cfg.tokens
    dy = make_dy(T, cfg.d_out, cfg.dtype, device="cuda")
    # the cached table is an input: the oracle's own top-k (fp64 logits), 3 % rows replaced
    fresh0 = O.topk_sorted(O.gate_logits(to_numpy64(g["x"]), to_numpy64(g["w_gate"])), k)
    cidx = np.ascontiguousarray(perturb_cached(fresh0, n, 0.03), dtype=np.int32)
    layer.set_cached_assignment(torch.from_numpy(cidx).cuda())
    y = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    rt = layer.routing(T)
    stats = layer.stats()
    h_buf, base = rt["h_buf"], rt["base"]
    grads = layer.backward(dy)
    torch.cuda.synchronize()
    assert layer.check_flags()[1] == 0
    lg = rt["logits"].cpu().double().numpy()
    fresh = O.topk_sorted(lg, k)
    assert np.array_equal(rt["fresh_idx"].cpu().numpy(), fresh)
    assert np.array_equal(rt["idx"].cpu().numpy(), cidx)
    ort = O.route(cidx, caps, n)
    assert np.array_equal(rt["slot_of"].cpu().numpy(), ort.slot_of)
    hits = int((np.sort(fresh, axis=1) == np.sort(cidx, axis=1)).all(axis=1).sum())
    assert stats["hit_count"] == hits and 0 < hits < T
    rb = layer.routing(T)
    dl, dw = rb["dl"].cpu().double().numpy(), rb["dw"].cpu().double().numpy()
    w = rt["w"].cpu().double().numpy()
    tol = TOL[cfg.dtype]
    rng = np.random.default_rng(5)
    stale = np.where((fresh != cidx).any(axis=1) & (ort.slot_of >= 0).all(axis=1))[0]
    samples = _samples(ort, T, k) + sorted(int(t) for t in rng.choice(stale, 4, replace=False))
    samples = sorted(set(samples))
    h_rows = {(t, r): h_buf[base[int(cidx[t, r])] + int(ort.slot_of[t, r])].float().cpu().numpy()
              for t in samples for r in range(k) if ort.slot_of[t, r] >= 0}
    kept = [t for t in samples if (ort.slot_of[t] >= 0).all()]
    dropped = [t for t in samples if (ort.slot_of[t] < 0).all()]
    for grp in (kept, dropped):
        st, gr = _group_oracle(cfg, g, grp, lg, cidx, ort.slot_of, h_rows, dy, cached=True)
        for j, t in enumerate(grp):
            assert rel(w[t], st.w[j]) <= 1e-5, t
            assert rel(to_numpy64(y[t]), st.y[j]) <= tol, t
            assert rel(dw[t], gr["dw"][j]) <= tol, t
            assert rel(dl[t], gr["dl"][j]) <= tol, t
            assert rel(to_numpy64(grads["dx"][t]), gr["dx"][j]) <= tol, t


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
