"""Pins for the fp64 oracle (run with -m "not gpu").

Each test ties the oracle to something other than itself: the paper/SPEC worked
examples, hand arithmetic, closed forms (dense mixture, plain MLP through torch
autograd), finite differences, brute-force definitions and invariants.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import moe_oracle as O


def _params(rng, n, d, f, d_out, scale=1.0):
    return dict(
        w_gate=rng.standard_normal((n, d)) * scale,
        w1=rng.standard_normal((n, f, d)) / math.sqrt(d),
        b1=rng.standard_normal((n, f)) * 0.3,
        w2=rng.standard_normal((n, d_out, f)) / math.sqrt(f),
        b2=rng.standard_normal((n, d_out)) * 0.3,
    )


def sig(z):
    return 1.0 / (1.0 + math.exp(-z))


# ----------------------------------------------------------------------------- Eq. 4
def test_capacity_spec_examples():
    # S:142-144 (Eq. 4)
    assert O.expert_capacity(1.0, 512, 2, 8) == 128
    assert O.expert_capacity(7.0, 64, 1, 4) == 112
    assert O.expert_capacity(1.25, 10, 1, 4) == 4
    assert O.expert_capacity(0.001, 10, 1, 4) == 1          # minimum 1
    assert O.capacities_from_factors([1.0, 2.0], 8, 1) == [4, 8]


# ----------------------------------------------------------------------------- softmax / top-k
def test_softmax_spec_examples():
    # S:59-60
    assert np.allclose(O.softmax(np.zeros((1, 4))), 0.25, atol=0, rtol=0)
    p = O.softmax(np.array([[1000.0, 0.0]]))
    assert np.isfinite(p).all() and p[0, 0] == 1.0 and p[0, 1] < 1e-300


def test_topk_spec_example():
    # scores [0.1,0.5,0.2,0.2], k=2 -> idx [1,2] (tie -> lower index), w [5/7, 2/7]
    l = np.log(np.array([[0.1, 0.5, 0.2, 0.2]]))
    assert l[0, 2] == l[0, 3]
    idx = O.topk(l, 2)
    assert idx.tolist() == [[1, 2]]
    w = O.gate_weights(l, idx, 1)
    assert abs(w[0, 0] - 5 / 7) < 1e-12 and abs(w[0, 1] - 2 / 7) < 1e-12
    # k = n: weights equal the input row (already sums to 1)
    idx4 = O.topk(l, 4)
    w4 = O.gate_weights(l, idx4, 1)
    assert np.allclose(w4[0], np.array([0.1, 0.5, 0.2, 0.2])[idx4[0]], atol=1e-12)
    # k = 1: weight exactly 1.0
    assert O.gate_weights(l, O.topk(l, 1), 1)[0, 0] == 1.0
    with pytest.raises(ValueError):
        O.topk(l, 5)


def test_topk_raw_mode_is_softmax_prob():
    l = np.array([[0.0, math.log(3.0)]])
    w = O.gate_weights(l, O.topk(l, 1), 0)
    assert abs(w[0, 0] - 0.75) < 1e-12


def test_topk_loop_matches_stable_sort_and_ties():
    rng = np.random.default_rng(0)
    for trial in range(20):
        n = int(rng.integers(2, 12))
        k = int(rng.integers(1, n + 1))
        l = rng.integers(-1, 2, size=(30, n)).astype(np.float64)   # tie-heavy
        if trial % 2:
            l = rng.standard_normal((30, n))
        a = O.topk(l, k)
        b = O.topk_sorted(l, k)
        assert (a == b).all()
        # definition: chosen set has no unchosen larger value, and among equals lower index wins
        for t in range(30):
            chosen = set(a[t].tolist())
            for e in range(n):
                if e in chosen:
                    continue
                for c in chosen:
                    assert l[t, e] < l[t, c] or (l[t, e] == l[t, c] and e > c)
    # -0.0 == +0.0 is a tie: lower index wins whichever sign it carries
    l = np.array([[0.0, -0.0, -1.0], [-0.0, 0.0, -1.0]])
    assert O.topk(l, 1).tolist() == [[0], [0]]
    assert O.topk_sorted(l, 1).tolist() == [[0], [0]]
    with pytest.raises(ValueError):
        O.topk(np.array([[np.nan, 1.0]]), 1)


# ----------------------------------------------------------------------------- GroupBy / drops
def test_groupby_spec_examples():
    # batch 4, k=1, assignments [0,1,0,1]
    idx = np.array([[0], [1], [0], [1]], np.int32)
    r = O.route(idx, [2, 2], 2)
    assert r.drops == 0 and r.slot_of[:, 0].tolist() == [0, 0, 1, 1]
    assert r.token_of_slot == [[0, 2], [1, 3]]
    r = O.route(idx, [1, 2], 2)
    assert r.drops == 1 and r.slot_of[:, 0].tolist() == [0, 0, -1, 1]   # (s2, rank 0) dropped


def test_route_matches_bruteforce_and_invariants():
    rng = np.random.default_rng(1)
    for trial in range(30):
        n = int(rng.integers(1, 9))
        k = int(rng.integers(1, n + 1))
        T = int(rng.integers(0, 40))
        idx = np.array([rng.permutation(n)[:k] for _ in range(T)], np.int32).reshape(T, k)
        caps = [int(c) for c in rng.integers(1, 12, size=n)]
        r = O.route(idx, caps, n)
        assert (r.slot_of == O.route_bruteforce(idx, caps, n)).all()
        assert r.counts.sum() == T * k                                  # conservation
        assert r.kept.sum() == T * k - r.drops
        for e in range(n):
            assert r.kept[e] == min(r.counts[e], caps[e])
            ids = r.token_of_slot[e]
            assert ids == sorted(ids) and len(set(ids)) == len(ids)     # increasing token ids
            assert len(ids) == r.kept[e]
            for s, code in enumerate(ids):                               # inverse maps
                assert r.slot_of[code // k, code % k] == s
            # each over-full expert drops exactly its (cnt - C) highest token ids
            all_t = [t for t in range(T) if e in idx[t]]
            dropped = [t for t in all_t if r.slot_of[t, list(idx[t]).index(e)] < 0]
            assert dropped == all_t[caps[e]:]


def test_route_ep_split_equals_single():
    # reading 12: global capacity over T_g, R-rank routing equals 1-rank routing
    rng = np.random.default_rng(2)
    n, k, T = 5, 2, 24
    idx = np.stack([rng.permutation(n)[:k] for _ in range(T)]).astype(np.int32)
    caps = [7, 3, 12, 9, 4]
    one = O.route(idx, caps, n)
    prior = np.zeros(n, np.int64)
    for lo, hi in [(0, 10), (10, 17), (17, 24)]:
        part = O.route(idx[lo:hi], caps, n, token_offset=lo, prior_counts=prior)
        assert (part.slot_of == one.slot_of[lo:hi]).all()
        prior = prior + part.counts


# ----------------------------------------------------------------------------- worked example
def _worked(golden_dir):
    with open(os.path.join(golden_dir, "worked_example.json")) as fh:
        g = json.load(fh)
    params = dict(
        w_gate=np.array(g["w_gate"], float),
        w1=np.stack([np.eye(2)] * 3),
        b1=np.array([[-0.5, 0.0]] * 3),
        w2=np.stack([(e + 1) * np.eye(2) for e in range(3)]),
        b2=np.array([[e, 0.0] for e in range(3)], float),
    )
    return g, params


def test_worked_example_hand_values(golden_dir):
    g, params = _worked(golden_dir)
    st = O.moe_forward(np.array(g["x"], float), params, 2, [3, 2, 1], renormalize=1)
    # by hand: x0 -> experts 0,1 with weights sigma(1), sigma(-1);
    # E_0(x0) = 1*relu([0.5, 0]) + [0,0]; E_1(x0) = 2*relu([0.5,0]) + [1,0] = [2, 0]
    assert abs(st.y[0, 0] - (sig(1) * 0.5 + sig(-1) * 2.0)) < 1e-12
    assert abs(st.w[3, 0] - sig(2)) < 1e-12
    assert st.y[3].tolist() == [0.0, 0.0]                 # fully dropped token


@pytest.mark.parametrize("case", ["case_A", "case_B"])
def test_worked_example_golden(golden_dir, case):
    g, params = _worked(golden_dir)
    c = g[case]
    x = np.array(g["x"], float)
    st = O.moe_forward(x, params, 2, c["capacities"], renormalize=1)
    assert np.array_equal(st.logits, np.array(g["logits"], float))
    assert st.idx.tolist() == g["idx"]
    assert np.allclose(st.w, g["w"], atol=1e-9)
    assert st.routing.counts.tolist() == g["counts"]
    gr = O.moe_backward(st, np.array(g["dy"], float))
    tol = 1e-9
    if case == "case_A":
        assert st.routing.slot_of.tolist() == c["slot_of"] and st.routing.drops == c["drops"]
        for key in ["y"]:
            assert np.allclose(st.y, c[key], atol=tol)
        assert np.allclose(gr["dw"], c["dw"], atol=tol)
        assert np.allclose(gr["dl"], c["dl"], atol=tol)
        assert np.allclose(gr["dx"], c["dx"], atol=tol)
        assert np.allclose(gr["dw_gate"], c["dw_gate"], atol=tol)
        for e in (0, 2):
            ex = c[f"expert{e}"]
            assert np.allclose(gr["dw1"][e], ex["dw1"], atol=tol)
            assert np.allclose(gr["db1"][e], ex["db1"], atol=tol)
            assert np.allclose(gr["dw2"][e], ex["dw2"], atol=tol)
            assert np.allclose(gr["db2"][e], ex["db2"], atol=tol)
    else:
        assert st.routing.slot_of[3].tolist() == c["slot_of_t3"]
        assert np.allclose(st.y[3], c["y_t3"], atol=tol)
        assert np.allclose(gr["dw"][3], c["dw_t3"], atol=tol)
        assert np.allclose(gr["dl"][3], c["dl_t3"], atol=tol)   # dropped e0 still gets gradient
        assert np.allclose(gr["dx"][3], c["dx_t3"], atol=tol)   # pins relu'(0) = 0
        assert np.allclose(gr["dw_gate"][:, 0], c["dw_gate_col0"], atol=tol)
        ex = c["expert1"]
        assert np.allclose(gr["dw1"][1], ex["dw1"], atol=tol)
        assert np.allclose(gr["db1"][1], ex["db1"], atol=tol)
        assert np.allclose(gr["dw2"][1], ex["dw2"], atol=tol)
        assert np.allclose(gr["db2"][1], ex["db2"], atol=tol)


# ----------------------------------------------------------------------------- closed forms
def test_aggregate_special_cases():
    rng = np.random.default_rng(3)
    T, d, f = 9, 5, 7
    x = rng.standard_normal((T, d))
    p = _params(rng, 1, d, f, d)
    st = O.moe_forward(x, p, 1, [T], renormalize=1)          # n = 1 -> identity aggregate
    H = np.maximum(x @ p["w1"][0].T + p["b1"][0], 0)
    assert np.allclose(st.y, H @ p["w2"][0].T + p["b2"][0], atol=1e-12)
    # two experts with identical parameters -> y equals that expert's output
    p2 = _params(rng, 2, d, f, d)
    for key in ("w1", "b1", "w2", "b2"):
        p2[key][1] = p2[key][0]
    st = O.moe_forward(x, p2, 2, [T, T], renormalize=1)
    H = np.maximum(x @ p2["w1"][0].T + p2["b1"][0], 0)
    assert np.allclose(st.y, H @ p2["w2"][0].T + p2["b2"][0], atol=1e-12)


@pytest.mark.parametrize("renorm", [0, 1])
def test_dense_mixture_closed_form(renorm):
    # k = n, C >= T: y = sum_e w_e FFN_e(x), computed with einsum over all experts
    rng = np.random.default_rng(4)
    n, T, d, f, do = 4, 11, 6, 8, 5
    x = rng.standard_normal((T, d))
    p = _params(rng, n, d, f, do)
    st = O.moe_forward(x, p, n, [T] * n, renormalize=renorm)
    l = x @ p["w_gate"].T
    pr = np.exp(l - l.max(1, keepdims=True)); pr /= pr.sum(1, keepdims=True)
    H = np.maximum(np.einsum("td,efd->tef", x, p["w1"]) + p["b1"][None], 0)
    Oall = np.einsum("tef,eof->teo", H, p["w2"]) + p["b2"][None]
    y = np.einsum("te,teo->to", pr, Oall)                   # renorm over all n == softmax
    assert np.allclose(st.y, y, atol=1e-12)


def test_single_expert_is_plain_mlp_autograd():
    # n = 1, k = 1, C >= T: the layer is a plain MLP; gradients via torch autograd in fp64
    rng = np.random.default_rng(5)
    T, d, f, do = 13, 6, 9, 4
    x = rng.standard_normal((T, d))
    p = _params(rng, 1, d, f, do)
    dy = rng.standard_normal((T, do))
    st = O.moe_forward(x, p, 1, [T], renormalize=0)
    gr = O.moe_backward(st, dy)
    tx = torch.tensor(x, requires_grad=True)
    tw1 = torch.tensor(p["w1"][0], requires_grad=True)
    tb1 = torch.tensor(p["b1"][0], requires_grad=True)
    tw2 = torch.tensor(p["w2"][0], requires_grad=True)
    tb2 = torch.tensor(p["b2"][0], requires_grad=True)
    twg = torch.tensor(p["w_gate"], requires_grad=True)
    pg = torch.softmax(tx @ twg.T, dim=1)[:, 0:1]             # raw mode, n=1: p == 1
    y = pg * (torch.relu(tx @ tw1.T + tb1) @ tw2.T + tb2)
    (y * torch.tensor(dy)).sum().backward()
    assert np.allclose(st.y, y.detach().numpy(), atol=1e-12)
    assert np.allclose(gr["dx"], tx.grad.numpy(), atol=1e-12)
    assert np.allclose(gr["dw1"][0], tw1.grad.numpy(), atol=1e-12)
    assert np.allclose(gr["db1"][0], tb1.grad.numpy(), atol=1e-12)
    assert np.allclose(gr["dw2"][0], tw2.grad.numpy(), atol=1e-12)
    assert np.allclose(gr["db2"][0], tb2.grad.numpy(), atol=1e-12)
    assert np.allclose(gr["dw_gate"], twg.grad.numpy(), atol=1e-12)


# ----------------------------------------------------------------------------- finite differences
def _fd_case(n, k, renorm, caps_scale, seed):
    rng = np.random.default_rng(seed)
    T, d, f, do = 8, 4, 5, 3
    for _ in range(200):
        x = rng.standard_normal((T, d))
        p = _params(rng, n, d, f, do, scale=1.0)
        l = x @ p["w_gate"].T
        s = np.sort(l, axis=1)
        if (np.diff(s, axis=1).min() < 1e-3):
            continue
        st = O.moe_forward(x, p, k, [max(1, int(T * caps_scale))] * n, renorm)
        if min((np.abs(a).min() if a.size else 1.0) for a in st.A) < 1e-3:
            continue
        return x, p, st, rng.standard_normal((T, do))
    raise RuntimeError("no well-separated draw")


@pytest.mark.parametrize("n,k", [(4, 1), (4, 2), (8, 2)])
@pytest.mark.parametrize("renorm", [0, 1])
@pytest.mark.parametrize("caps_scale", [1.0, 0.25])
def test_finite_differences(n, k, renorm, caps_scale):
    # central differences, h = 1e-6, rel 1e-4; caps_scale 0.25 forces drops
    x, p, st, dy = _fd_case(n, k, renorm, caps_scale, seed=10 * n + k + renorm)
    caps = st.capacities
    gr = O.moe_backward(st, dy)

    def loss(xx, pp):
        s2 = O.moe_forward(xx, pp, k, caps, renorm)
        assert (s2.idx == st.idx).all() and (s2.routing.slot_of == st.routing.slot_of).all()
        return float((s2.y * dy).sum())

    h = 1e-6
    rng = np.random.default_rng(99)
    checks = [("x", None)] + [(key, key) for key in ("w_gate", "w1", "b1", "w2", "b2")]
    for name, key in checks:
        base = x if key is None else p[key]
        g = gr["dx"] if key is None else gr[{"w_gate": "dw_gate", "w1": "dw1", "b1": "db1",
                                             "w2": "dw2", "b2": "db2"}[key]]
        flat_idx = rng.choice(base.size, size=min(6, base.size), replace=False)
        num = []
        for fi in flat_idx:
            ii = np.unravel_index(fi, base.shape)
            plus = base.copy(); plus[ii] += h
            minus = base.copy(); minus[ii] -= h
            if key is None:
                fp, fm = loss(plus, p), loss(minus, p)
            else:
                pp = dict(p); pp[key] = plus; fp = loss(x, pp)
                pm = dict(p); pm[key] = minus; fm = loss(x, pm)
            num.append((fp - fm) / (2 * h))
        num = np.array(num)
        ana = g.reshape(-1)[flat_idx]
        scale = max(np.abs(g).max(), 1e-8)
        assert np.abs(num - ana).max() / scale < 1e-4, (name, num, ana)


# ----------------------------------------------------------------------------- equivalences
def test_cached_equals_uncached_when_hit():
    # cached = fresh top-k -> identical routing and outputs; hit_count = T
    rng = np.random.default_rng(6)
    n, k, T, d, f = 6, 2, 40, 5, 7
    x = rng.standard_normal((T, d))
    p = _params(rng, n, d, f, d)
    caps = [9] * n
    a = O.moe_forward(x, p, k, caps, 1)
    b = O.moe_forward(x, p, k, caps, 1, cached_idx=a.fresh_idx.copy())
    assert b.hit_count == T and np.array_equal(a.y, b.y)
    # reversed r order is the same set: still a hit, weights follow the supplied order
    c = O.moe_forward(x, p, k, caps, 1, cached_idx=a.fresh_idx[:, ::-1].copy())
    assert c.hit_count == T
    assert np.allclose(c.w, a.w[:, ::-1], atol=1e-15)
    # a stale row: routed to the stale experts with fresh weights
    stale = a.fresh_idx.copy()
    stale[0] = [e for e in range(n) if e not in stale[0]][:k]
    d_ = O.moe_forward(x, p, k, caps, 1, cached_idx=stale)
    assert d_.hit_count == T - 1
    lsel = d_.logits[0, stale[0]]
    wexp = np.exp(lsel - lsel.max()); wexp /= wexp.sum()
    assert np.allclose(d_.w[0], wexp, atol=1e-15)
    with pytest.raises(ValueError):
        bad = a.fresh_idx.copy(); bad[0] = [0, 0]
        O.moe_forward(x, p, k, caps, 1, cached_idx=bad)


def test_assignment_cache_spec_examples():
    """SPEC cache_step / cached_route examples."""
    rng = np.random.default_rng(9)
    n, k, T, d, f, N = 6, 2, 30, 5, 7, 50
    x = rng.standard_normal((T, d))
    p = _params(rng, n, d, f, d)
    caps = [T] * n
    ids = rng.permutation(N)[:T]
    cache = O.AssignmentCache(N, k)
    a = O.moe_forward(x, p, k, caps, 1)
    # first epoch: empty cache -> hit fraction 0.0 by convention, every sample falls back
    assert cache.hit_fraction(ids, a.fresh_idx) == 0.0
    assert not cache.known(ids).any()
    idx = cache.lookup(ids, a.fresh_idx)
    assert np.array_equal(idx, a.fresh_idx)
    b = O.moe_forward(x, p, k, caps, 1, cached_idx=np.full((T, k), -1), cache_fallback=True)
    assert b.hit_count == 0 and np.array_equal(b.y, a.y)     # fallback = uncached routing
    cache.update(ids, a.fresh_idx)
    # identical assignments across epochs -> hit fraction 1.0, bit-identical outputs
    assert cache.hit_fraction(ids, a.fresh_idx) == 1.0
    c = O.moe_forward(x, p, k, caps, 1, cached_idx=cache.lookup(ids, a.fresh_idx))
    assert c.hit_count == T and np.array_equal(c.y, a.y)
    # all samples reassigned -> 0.0
    other = np.array([[e for e in range(n) if e not in row][:k] for row in a.fresh_idx], np.int32)
    cache.update(ids, other)
    assert cache.hit_fraction(ids, a.fresh_idx) == 0.0
    # one unknown sample among known ones: it is routed by its fresh top-k and is a miss;
    # the others use the remembered rows
    cache.update(ids, a.fresh_idx)
    cache.table[ids[3]] = -1
    rows = cache.table[ids].copy()
    e_ = O.moe_forward(x, p, k, caps, 1, cached_idx=rows, cache_fallback=True)
    assert e_.hit_count == T - 1
    assert np.array_equal(e_.idx, a.fresh_idx) and np.array_equal(e_.y, a.y)
    # without the fallback an unknown row is an error (v1 contract)
    with pytest.raises(ValueError):
        O.moe_forward(x, p, k, caps, 1, cached_idx=rows)


def test_capacity_change_without_drops_is_identity():
    # S:158 plan equivalence
    rng = np.random.default_rng(7)
    n, k, T, d, f = 5, 2, 30, 4, 6
    x = rng.standard_normal((T, d))
    p = _params(rng, n, d, f, d)
    a = O.moe_forward(x, p, k, [T] * n, 1)
    b = O.moe_forward(x, p, k, [int(c) for c in a.routing.counts], 1)
    assert a.routing.drops == 0 and b.routing.drops == 0
    assert np.array_equal(a.y, b.y)


# ----------------------------------------------------------------------------- policies
def test_capacity_policy_traces():
    n, Tg, k = 4, 400, 1
    # constant balanced trace: settles, then no recompile storm
    pol = O.CapacityPolicy(n, Tg, k, [100] * n)
    changes = [pol.update([100] * n) for _ in range(60)]
    assert sum(c is not None for c in changes[25:]) == 0
    # step trace: one expert doubles -> grows within one evaluation, others unchanged
    pol = O.CapacityPolicy(n, Tg, k, [115] * n)
    for _ in range(5):
        assert pol.update([100] * n) is None                     # hysteresis
    new = pol.update([200, 100, 100, 100])
    assert new is not None and new[0] == math.ceil(1.15 * 200) and new[1:] == [115] * 3
    # shrink only after a full window of low utilisation
    pol = O.CapacityPolicy(n, Tg, k, [400] * n)
    outs = [pol.update([50] * n) for _ in range(20)]
    assert all(o is None for o in outs[:19]) and outs[19] == [math.ceil(1.15 * 50)] * n
    # clamp to alpha in [0.25, 8]
    pol = O.CapacityPolicy(n, Tg, k, [100] * n, max_alpha=2.0)
    new = pol.update([1000, 0, 0, 0])
    assert new[0] == O.expert_capacity(2.0, Tg, k, n)


def test_caching_trigger_spec_examples():
    # S:461-464
    assert O.caching_trigger(0.99, 5, False) is False
    assert O.caching_trigger(0.97, 12, False) is True
    assert O.caching_trigger(0.88, 48, True) is False
    for h in np.linspace(0.905, 0.955, 11):                    # hysteresis band
        assert O.caching_trigger(h, 20, True) is True
        assert O.caching_trigger(h, 20, False) is False


def test_round_bf16_matches_torch():
    rng = np.random.default_rng(8)
    a = np.concatenate([rng.standard_normal(10000) * 10.0 ** rng.integers(-5, 5, 10000),
                        np.array([0.0, -0.0, 1.0, 1.00390625, 1.01171875])])
    ref = torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(O.round_bf16(a), ref)


# ----------------------------------------------------------------------------- N3: loss variants
def test_balance_term_spec_examples():
    # S:329-332 (Eq. 3)
    lam = 0.37
    n = 4
    assert abs(O.balance_term([1 / n] * n, [1 / n] * n, lam) - lam) < 1e-15      # uniform -> lambda
    assert abs(O.balance_term([1, 0, 0, 0], [1, 0, 0, 0], lam) - 4 * lam) < 1e-15  # collapse -> n lambda
    assert abs(O.balance_term([0.5, 0.5], [0.6, 0.4], 0.01) - 0.01) < 1e-15
    # fractions: T sums to 1 over the T*k assignments, G sums to 1
    rng = np.random.default_rng(11)
    l = rng.standard_normal((50, 6))
    idx = O.topk(l, 2)
    Tf, Gf = O.balance_fractions(O.route(idx, [50] * 6, 6).counts, O.softmax(l), 2)
    assert abs(Tf.sum() - 1) < 1e-12 and abs(Gf.sum() - 1) < 1e-12


def test_aggregate_spec_special_cases():
    rng = np.random.default_rng(12)
    n, T, d, f = 3, 12, 4, 5
    x = rng.standard_normal((T, d))
    p = _params(rng, n, d, f, d)
    st = O.moe_forward(x, p, 1, [T] * n, 1)
    spec, valid = st.extra["spec"], st.extra["spec_valid"]
    # k = 1, no drops: spec rows are the de-grouped expert predictions; with w = 1 == y
    assert valid.all() and np.allclose(spec, st.y, atol=1e-12)
    st2 = O.moe_forward(x, p, 2, [2] * n, 1)                   # drops -> invalid zero rows
    sp2, v2 = st2.extra["spec"], st2.extra["spec_valid"]
    assert (v2 == (st2.routing.slot_of.reshape(-1) >= 0)).all()
    assert np.abs(sp2[v2 == 0]).max() == 0.0
    # weighted sum of the valid spec rows reproduces y (Eq. 1 inner sum vs Eq. 2 rows)
    w = st2.w.reshape(-1, 1)
    assert np.allclose((sp2 * w).reshape(T, 2, d).sum(1), st2.y, atol=1e-12)


@pytest.mark.parametrize("renorm", [0, 1])
def test_loss_variants_finite_differences(renorm):
    """L = sum(dy*y) + sum(c*spec) + sum(cw*w) + B(lambda): analytic vs central differences."""
    n, k, lam = 4, 2, 0.3
    x, p, st, dy = _fd_case(n, k, renorm, 1.0, seed=77)
    rng = np.random.default_rng(78)
    T = x.shape[0]
    cs = rng.standard_normal((T * k, dy.shape[1]))
    cw = rng.standard_normal((T, k))
    caps = st.capacities

    def full(xx, pp):
        s2 = O.moe_forward(xx, pp, k, caps, renorm, balance_lambda=lam)
        assert (s2.idx == st.idx).all()
        return s2, float((s2.y * dy).sum() + (s2.extra["spec"] * cs).sum() + (s2.w * cw).sum()
                         + s2.extra["aux_loss"])

    s0, _ = full(x, p)
    gr = O.moe_backward(s0, dy, dspec=cs, dw_ext=cw)
    h = 1e-6
    for key, gk in (("w_gate", "dw_gate"), ("w1", "dw1"), ("b2", "db2")):
        base = p[key]
        for fi in np.random.default_rng(5).choice(base.size, 5, replace=False):
            ii = np.unravel_index(fi, base.shape)
            pp = dict(p); pl = base.copy(); pl[ii] += h; pp[key] = pl
            pm = dict(p); mi = base.copy(); mi[ii] -= h; pm[key] = mi
            num = (full(x, pp)[1] - full(x, pm)[1]) / (2 * h)
            ana = gr[gk][ii]
            assert abs(num - ana) <= 1e-4 * max(1.0, np.abs(gr[gk]).max()), (key, num, ana)
    for fi in range(0, x.size, 7):
        ii = np.unravel_index(fi, x.shape)
        xp = x.copy(); xp[ii] += h
        xm = x.copy(); xm[ii] -= h
        num = (full(xp, p)[1] - full(xm, p)[1]) / (2 * h)
        assert abs(num - gr["dx"][ii]) <= 1e-4 * max(1.0, np.abs(gr["dx"]).max())


def test_relu_mask_argument():
    """relu_mask (the kernel's ReLU' decisions): the mask A > 0 reproduces the
    default gradients exactly, and flipping one decision changes exactly that dA element --
    dx / dW1 / db1 of its expert move by the outer products the chain rule predicts."""
    x, p, st, dy = _fd_case(4, 2, 1, 1.0, 5)
    g0 = O.moe_backward(st, dy)
    g1 = O.moe_backward(st, dy, relu_mask=[a > 0 for a in st.A])
    for kk in ("dx", "dw_gate", "dw1", "db1", "dw2", "db2", "dl"):
        assert np.array_equal(g0[kk], g1[kk]), kk
    e = max(range(len(st.A)), key=lambda j: st.A[j].shape[0])
    mask = [a > 0 for a in st.A]
    r, c = 0, int(np.argmax(st.A[e][0] > 0))
    assert st.A[e][r, c] > 0
    mask[e] = mask[e].copy()
    mask[e][r, c] = False
    g2 = O.moe_backward(st, dy, relu_mask=mask)
    W2 = np.asarray(p["w2"][e], np.float64)
    W1 = np.asarray(p["w1"][e], np.float64)
    dA_rc = float(g0["dO"][e][r] @ W2[:, c])          # the element the flip removes
    assert math.isclose(g0["db1"][e][c] - g2["db1"][e][c], dA_rc, rel_tol=1e-12, abs_tol=1e-15)
    want_dW1 = np.zeros_like(g0["dw1"][e])
    want_dW1[c] = dA_rc * st.X[e][r]
    assert np.allclose(g0["dw1"][e] - g2["dw1"][e], want_dW1, rtol=1e-12, atol=1e-15)
    assert np.allclose(g0["dX"][e][r] - g2["dX"][e][r], dA_rc * W1[c], rtol=1e-12, atol=1e-15)
    others = [j for j in range(len(st.A)) if j != e]
    for j in others:
        assert np.array_equal(g0["dw1"][j], g2["dw1"][j])
    assert np.array_equal(g0["dw2"], g2["dw2"])
