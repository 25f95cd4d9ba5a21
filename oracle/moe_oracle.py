"""Plain, slow, fp64 CPU oracle of the DynaMoE MoE-layer hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this module.  The product path
(paper_2205_01848_b200/) never imports it and shares no code with it.

Every function cites the PAPER.md passage (P:line) it follows; readings of
points the paper leaves open are SURVEY.md §8(c) readings 1-15 and are listed in
DESIGN.md §"Readings".  Arithmetic is NumPy float64 unless a function says
otherwise; routing is integer loops.  There is no blocking, fusion or reordering
beyond the definitions: a reader can check each step against Alg. 1,
Eq. 4, the drop rule and the caching description.

Pins (tests/test_oracle.py): the hand-checkable worked example (tests/golden/),
SPEC's worked examples, central
finite differences of the whole layer, the dense-mixture closed form (k = n, no
drops), the n = 1 plain-MLP closed form via torch autograd, a brute-force
routing definition, and the conservation / drop-order invariants.
Functions without a pin: none (the capacity policy is pinned only by synthetic
traces, because the paper gives no policy - reading 14).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


# --------------------------------------------------------------------------- #
# Eq. 4: expert capacity  C = alpha * batch_size * k / n
# --------------------------------------------------------------------------- #
def expert_capacity(alpha: float, tokens_global: int, k: int, n: int) -> int:
    """Eq. 4.  Reading 5: ceil, minimum 1, batch_size = global token count,
    computed in fp64 on the host."""
    return max(1, int(math.ceil(alpha * tokens_global * k / n)))


def capacities_from_factors(alphas, tokens_global: int, k: int) -> list[int]:
    """Per-expert capacity factors alpha_e (dynamic capacity factors)."""
    n = len(alphas)
    return [expert_capacity(float(a), tokens_global, k, n) for a in alphas]


# --------------------------------------------------------------------------- #
# Alg. 1 line 1: score <- G(x); reading 1: G is one linear layer, no bias
# --------------------------------------------------------------------------- #
def gate_logits(x: np.ndarray, w_gate: np.ndarray) -> np.ndarray:
    """l = x W_g^T  ([T,d] x [n,d]^T -> [T,n]), fp64."""
    return np.asarray(x, np.float64) @ np.asarray(w_gate, np.float64).T


def softmax(l: np.ndarray) -> np.ndarray:
    """Reading 2: score = softmax probabilities; row-max subtraction."""
    l = np.asarray(l, np.float64)
    m = l.max(axis=-1, keepdims=True)
    e = np.exp(l - m)
    return e / e.sum(axis=-1, keepdims=True)


# --------------------------------------------------------------------------- #
# Alg. 1 line 2: indices <- argmax_k(score)
# --------------------------------------------------------------------------- #
def topk(logits: np.ndarray, k: int) -> np.ndarray:
    """Reading 3: select on the logits (softmax is monotone); IEEE '>' comparison;
    equal values (including -0.0 == +0.0) go to the LOWER expert index; output
    column r is the r-th best.  Plain loop: repeatedly take the first maximum of
    the experts not yet taken.  NaN logits are rejected."""
    logits = np.asarray(logits)
    T, n = logits.shape
    if not (1 <= k <= n):
        raise ValueError("k must satisfy 1 <= k <= n (S:206)")
    if np.isnan(logits).any():
        raise ValueError("NaN logit")
    idx = np.empty((T, k), np.int32)
    for t in range(T):
        taken = [False] * n
        for r in range(k):
            best = -1
            for e in range(n):
                if taken[e]:
                    continue
                if best < 0 or logits[t, e] > logits[t, best]:
                    best = e
            taken[best] = True
            idx[t, r] = best
    return idx


def topk_sorted(logits: np.ndarray, k: int) -> np.ndarray:
    """Same rule as `topk`, vectorised: a stable argsort of -logits keeps equal values in
    ascending index order.  (-0.0 and +0.0 compare equal in the sort.)  Used to
    cross-check `topk` and for large T."""
    logits = np.asarray(logits, np.float64)
    if np.isnan(logits).any():
        raise ValueError("NaN logit")
    return np.argsort(-logits, axis=1, kind="stable")[:, :k].astype(np.int32)


# --------------------------------------------------------------------------- #
# Alg. 1 line 3: (w_1..w_k) <- normalize(score[indices])
# --------------------------------------------------------------------------- #
def gate_weights(logits: np.ndarray, idx: np.ndarray, renormalize: int) -> np.ndarray:
    """Reading 4.  renormalize=1: w_r = p_{i_r} / sum_r' p_{i_r'}  (sum-normalisation of the
    selected softmax probabilities), evaluated as exp(l_{i_r} - m) / sum exp(l_{i_r'} - m)
    with m the largest selected logit (equal in exact arithmetic).  renormalize=0: w_r =
    p_{i_r} (raw softmax probability, Switch-style)."""
    logits = np.asarray(logits, np.float64)
    T, k = idx.shape
    w = np.empty((T, k), np.float64)
    if renormalize:
        for t in range(T):
            sel = logits[t, idx[t]]
            e = np.exp(sel - sel.max())
            w[t] = e / e.sum()
    else:
        p = softmax(logits)
        for t in range(T):
            w[t] = p[t, idx[t]]
    return w


# --------------------------------------------------------------------------- #
# GroupBy with capacity (Eq. 4, App. A)
# --------------------------------------------------------------------------- #
@dataclass
class Routing:
    counts: np.ndarray          # [n] pre-drop assignment counts cnt_e
    kept: np.ndarray            # [n] min(cnt_e, C_e)
    slot_of: np.ndarray         # [T,k] slot inside expert idx[t,r]'s buffer, -1 = dropped
    token_of_slot: list         # per expert: list of t_g*k + r for slots 0..kept_e-1
    drops: int


def route(idx: np.ndarray, capacities, n: int, token_offset: int = 0,
          prior_counts=None) -> Routing:
    """Capacity-bounded grouping.  P:225: samples that "still don't fit" are dropped.
    Reading 6 (token-major first fit): walk assignments in order
    (t ascending, then r ascending) over the global token index t_g = token_offset + t;
    pos = cnt_e; cnt_e += 1; kept iff pos < C_e.  `prior_counts` (EP, reading 12) are the
    assignments to each expert from tokens with smaller global index on other ranks."""
    T, k = idx.shape
    cnt = [0] * n if prior_counts is None else [int(c) for c in prior_counts]
    start = list(cnt)
    slot_of = np.full((T, k), -1, np.int32)
    tos = [[] for _ in range(n)]
    for t in range(T):
        for r in range(k):
            e = int(idx[t, r])
            pos = cnt[e]
            cnt[e] += 1
            if pos < capacities[e]:
                slot_of[t, r] = pos
                tos[e].append((token_offset + t) * k + r)
    counts = np.array([cnt[e] - start[e] for e in range(n)], np.int64)
    kept = np.array([max(0, min(cnt[e], capacities[e]) - min(start[e], capacities[e]))
                     for e in range(n)], np.int64)
    drops = int(counts.sum() - kept.sum())
    return Routing(counts, kept, slot_of, tos, drops)


def route_bruteforce(idx: np.ndarray, capacities, n: int):
    """Definition-level restatement used as a pin: pos(t,r) = #{(t',r') earlier in token-major
    order with idx[t',r'] == idx[t,r]}; kept iff pos < C_e."""
    T, k = idx.shape
    slot = np.full((T, k), -1, np.int32)
    for t in range(T):
        for r in range(k):
            e = idx[t, r]
            pos = int((idx[:t] == e).sum() + (idx[t, :r] == e).sum())
            if pos < capacities[e]:
                slot[t, r] = pos
    return slot


# --------------------------------------------------------------------------- #
# Expert FFN, Alg. 1 line 7 with reading 9 (2-layer ReLU MLP with biases)
# --------------------------------------------------------------------------- #
def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round fp64 values to the nearest bf16 (ties to even) via fp32, emulating the
    storage points of reading 10.  Used only when emulate_bf16=True."""
    f = np.asarray(a, np.float64).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def expert_ffn(X: np.ndarray, W1, b1, W2, b2, emulate_bf16=False):
    """A = X W1^T + b1; H = max(A, 0); O = H W2^T + b2 (torch Linear layout)."""
    A = X @ W1.T + b1
    H = np.maximum(A, 0.0)
    if emulate_bf16:
        H = round_bf16(H)
    O = H @ W2.T + b2
    if emulate_bf16:
        O = round_bf16(O)
    return A, H, O


# --------------------------------------------------------------------------- #
# Whole layer forward (Alg. 1) + capacity + caching
# --------------------------------------------------------------------------- #
@dataclass
class FwdState:
    x: np.ndarray
    params: dict
    k: int
    n: int
    capacities: list
    renormalize: int
    logits: np.ndarray
    p: np.ndarray
    idx: np.ndarray             # indices actually used for dispatch (cached or fresh)
    fresh_idx: np.ndarray       # fresh top-k of this step's gate
    w: np.ndarray
    routing: Routing
    X: list                     # per expert [C_e, d], rows >= kept_e zero
    A: list
    H: list
    O: list
    y: np.ndarray
    hit_count: int = 0
    emulate_bf16: bool = False
    token_offset: int = 0
    extra: dict = field(default_factory=dict)


# --------------------------------------------------------------------------- #
# Eq. 3 balance term and the AggregateSpec output (App. A)
# --------------------------------------------------------------------------- #
def balance_term(T_frac, G_frac, lam: float) -> float:
    """Eq. 3: B = lambda * n * sum_i T_i * G_i (n = len(T_frac))."""
    T_frac = np.asarray(T_frac, np.float64)
    return float(lam * len(T_frac) * np.sum(T_frac * np.asarray(G_frac, np.float64)))


def balance_fractions(counts_pre, p, k: int):
    """T_i: fraction of the (token, slot) assignments routed to expert i, PRE-drop counts
    (S:347-348), normalised over the batch's T*k assignments (S:186 'count_i / (batch*k)');
    G_i: mean gate probability of expert i over the batch."""
    p = np.asarray(p, np.float64)
    return np.asarray(counts_pre, np.float64) / (p.shape[0] * k), p.mean(axis=0)


def aggregate_spec(O, idx, slot_of):
    """AggregateSpec (App. A): row t*k + r holds O_{idx[t,r]}[slot] -- the
    prediction of the r-th chosen expert for sample t -- or zeros with valid = 0 when the
    pair was dropped."""
    T, k = idx.shape
    d_out = next((o.shape[1] for o in O if o.ndim == 2), 0)
    out = np.zeros((T * k, d_out))
    valid = np.zeros(T * k, np.uint8)
    for t in range(T):
        for r in range(k):
            s = slot_of[t, r]
            if s >= 0:
                out[t * k + r] = O[idx[t, r]][s]
                valid[t * k + r] = 1
    return out, valid


class AssignmentCache:
    """Per-sample assignment cache (SPEC cache_step S:252-257 and cached_route
    S:259-267; reading 11): row s = the expert indices sample s was routed to the last time
    the gate saw it, -1 = unknown (never seen).

    lookup(): cached_route's dispatch indices for a batch: the remembered row of a known
    sample; for an unknown sample the fallback of S:263 ("falls back to gate-derived routing
    for that sample, counted as a miss"), i.e. the gate's fresh top-k.
    update(): cache_step's post-condition: after the gate's forward the remembered
    rows of the batch's samples are overwritten with the current (fresh) decision."""

    def __init__(self, num_samples: int, k: int):
        self.table = np.full((num_samples, k), -1, np.int32)

    def known(self, sample_ids):
        return np.array([bool((self.table[s] >= 0).all()) for s in sample_ids])

    def lookup(self, sample_ids, fresh):
        fresh = np.asarray(fresh, np.int32)
        idx = np.empty_like(fresh)
        for t, sid in enumerate(sample_ids):
            row = self.table[sid]
            idx[t] = row if (row >= 0).all() else fresh[t]
        return idx

    def hit_fraction(self, sample_ids, fresh):
        """fraction of the batch whose remembered row equals (as a set) the fresh
        decision; unknown samples are misses (first epoch -> 0.0)."""
        fresh = np.asarray(fresh)
        hits = 0
        for t, sid in enumerate(sample_ids):
            row = self.table[sid]
            if (row >= 0).all() and set(row.tolist()) == set(fresh[t].tolist()):
                hits += 1
        return hits / max(1, len(sample_ids))

    def update(self, sample_ids, fresh):
        fresh = np.asarray(fresh, np.int32)
        for t, sid in enumerate(sample_ids):
            self.table[sid] = fresh[t]


def moe_forward(x, params, k: int, capacities, renormalize: int = 1, cached_idx=None,
                logits=None, emulate_bf16: bool = False, token_offset: int = 0,
                prior_counts=None, balance_lambda: float = 0.0,
                cache_fallback: bool = False) -> FwdState:
    """One MoE layer forward.

    params: w_gate [n,d], w1 [n,f,d], b1 [n,f], w2 [n,d_out,f], b2 [n,d_out] (fp64 arrays).
    logits: if given (routing parity), these [T,n] values replace the
    fp64 gate logits for top-k, weights and backward; else l = x W_g^T.
    cached_idx: sample-assignment caching (reading 11): the cached [T,k] indices
    drive dispatch; weights are normalize(p[t, cached]) from the fresh gate; the fresh top-k
    is still computed and hit_count = #{t : set(fresh_t) == set(cached_t)}.
    cache_fallback: cached rows containing -1 are unknown samples: they are routed by the
    fresh top-k and counted as misses (AssignmentCache.lookup)."""
    x = np.asarray(x, np.float64)
    T = x.shape[0]
    wg = np.asarray(params["w_gate"], np.float64)
    n = wg.shape[0]
    l = gate_logits(x, wg) if logits is None else np.asarray(logits, np.float64)
    p = softmax(l)
    fresh = topk_sorted(l, k)
    if cached_idx is not None:
        idx = np.array(cached_idx, np.int32)
        known = np.ones(T, bool)
        for t in range(T):
            row = idx[t]
            if cache_fallback and (row < 0).any():
                idx[t] = fresh[t]          # unknown sample: gate-derived routing, a miss
                known[t] = False
                continue
            if len(set(row.tolist())) != k or row.min() < 0 or row.max() >= n:
                raise ValueError(f"invalid cached row {t}: {row}")
        hit = int(sum(known[t] and set(fresh[t].tolist()) == set(idx[t].tolist())
                      for t in range(T)))
    else:
        idx = fresh
        hit = 0
    w = gate_weights(l, idx, renormalize)
    rt = route(idx, capacities, n, token_offset, prior_counts)
    d = x.shape[1]
    X, A, H, O = [], [], [], []
    for e in range(n):
        Xe = np.zeros((capacities[e], d))            # zero-filled unused rows
        for j, code in enumerate(rt.token_of_slot[e]):
            t = code // k - token_offset
            Xe[j] = x[t]
        kept = int(rt.kept[e])
        Ae, He, Oe = expert_ffn(Xe[:kept], np.asarray(params["w1"][e], np.float64),
                                np.asarray(params["b1"][e], np.float64),
                                np.asarray(params["w2"][e], np.float64),
                                np.asarray(params["b2"][e], np.float64), emulate_bf16)
        X.append(Xe); A.append(Ae); H.append(He); O.append(Oe)
    d_out = np.asarray(params["w2"]).shape[1]
    y = np.zeros((T, d_out))
    # Alg. 1 lines 5-8: y += w_i * E_e(x), surviving pairs only, in r order
    for t in range(T):
        for r in range(k):
            s = rt.slot_of[t, r]
            if s >= 0:
                y[t] += w[t, r] * O[idx[t, r]][s]
    st = FwdState(x, params, k, n, list(capacities), renormalize, l, p, idx, fresh, w,
                  rt, X, A, H, O, y, hit, emulate_bf16, token_offset)
    st.extra["balance_lambda"] = float(balance_lambda)
    if balance_lambda:
        Tf, Gf = balance_fractions(rt.counts, p, k)
        st.extra["aux_loss"] = balance_term(Tf, Gf, balance_lambda)
        st.extra["T_frac"] = Tf
    st.extra["spec"], st.extra["spec_valid"] = aggregate_spec(O, idx, rt.slot_of)
    return st


# --------------------------------------------------------------------------- #
# Backward: exact chain rule of the forward above
# --------------------------------------------------------------------------- #
def moe_backward(st: FwdState, dy: np.ndarray, dspec=None, dw_ext=None, relu_mask=None) -> dict:
    """Gradients of sum(dy * y) w.r.t. x, w_gate, w1, b1, w2, b2 (and the logits, dl).

    P:225: dropped samples are ignored in back propagation -> dropped pairs get dw = 0 and
    no expert-gradient rows (reading 8).  Renorm mode: dl[t,i_r] = w_r (dw_r - sum w dw),
    zero for unselected experts; the dropped expert's logit still gets gradient through
    the renorm denominator.  Raw mode: dp_j = dw_r at j = i_r; dl = p (dp - <p,dp>).
    relu'(0) = 0 (reading 9).

    Optional loss variants (N3): dspec [T*k, d_out] is the gradient w.r.t. the AggregateSpec
    rows (specification loss, Eq. 2; rows of dropped pairs are ignored) and dw_ext
    [T, k] the caller's direct gradient w.r.t. the gate weights w (e.g. L_i of Eq. 2); the
    balance term (Eq. 3) adds dB/dl with T_i held constant (stop-gradient):
    dB/dp[t,i] = lambda n T_i / T.

    relu_mask: optional list over experts of boolean [kept_e x f] ReLU' decisions (H > 0 of
    the kernel under test).  The mask is an integer decision taken by floating point, so for
    parity both sides take it in the same precision (the kernel's, as the routing decisions
    come from the kernel's fp32 logits): an A within an ulp of 0 may otherwise flip sign
    between fp64 and fp32 and move a whole dA element.  None = A > 0 here."""
    dy = np.asarray(dy, np.float64)
    k, n = st.k, st.n
    T = st.x.shape[0]
    idx, w, rt = st.idx, st.w, st.routing
    d_out = dy.shape[1]
    dw = np.zeros((T, k))
    dO = [np.zeros((int(rt.kept[e]), d_out)) for e in range(n)]
    for t in range(T):
        for r in range(k):
            s = rt.slot_of[t, r]
            if s >= 0:
                e = idx[t, r]
                dO[e][s] = w[t, r] * dy[t]
                dw[t, r] = float(dy[t] @ st.O[e][s])
                if dspec is not None:
                    dO[e][s] = dO[e][s] + np.asarray(dspec, np.float64)[t * k + r]
                if dw_ext is not None:
                    dw[t, r] += float(dw_ext[t, r])
    if st.emulate_bf16:
        dO = [round_bf16(a) for a in dO]
    dW1 = np.zeros_like(np.asarray(st.params["w1"], np.float64))
    db1 = np.zeros_like(np.asarray(st.params["b1"], np.float64))
    dW2 = np.zeros_like(np.asarray(st.params["w2"], np.float64))
    db2 = np.zeros_like(np.asarray(st.params["b2"], np.float64))
    dX = []
    for e in range(n):
        kept = int(rt.kept[e])
        W1 = np.asarray(st.params["w1"][e], np.float64)
        W2 = np.asarray(st.params["w2"][e], np.float64)
        dW2[e] = dO[e].T @ st.H[e]
        db2[e] = dO[e].sum(axis=0)
        mask = (st.A[e] > 0) if relu_mask is None else np.asarray(relu_mask[e], bool)
        dA = (dO[e] @ W2) * mask
        if st.emulate_bf16:
            dA = round_bf16(dA)
        dW1[e] = dA.T @ st.X[e][:kept]
        db1[e] = dA.sum(axis=0)
        dX.append(dA @ W1)
    dl = np.zeros((T, n))
    if st.renormalize:
        for t in range(T):
            s = float(np.dot(w[t], dw[t]))
            for r in range(k):
                dl[t, idx[t, r]] = w[t, r] * (dw[t, r] - s)
    else:
        for t in range(T):
            dp = np.zeros(n)
            for r in range(k):
                dp[idx[t, r]] = dw[t, r]
            dl[t] = st.p[t] * (dp - float(np.dot(st.p[t], dp)))
    lam = st.extra.get("balance_lambda", 0.0)
    if lam:
        g = lam * n * st.extra["T_frac"] / T
        for t in range(T):
            dl[t] += st.p[t] * (g - float(np.dot(st.p[t], g)))
    wg = np.asarray(st.params["w_gate"], np.float64)
    dW_g = dl.T @ st.x
    dx = dl @ wg
    for t in range(T):
        for r in range(k):
            s = rt.slot_of[t, r]
            if s >= 0:
                dx[t] += dX[idx[t, r]][s]
    return dict(dx=dx, dw_gate=dW_g, dw1=dW1, db1=db1, dw2=dW2, db2=db2, dl=dl, dw=dw,
                dO=dO, dX=dX)


# --------------------------------------------------------------------------- #
# Dynamic capacity policy (reading 14 = SPEC S:449-456)
# --------------------------------------------------------------------------- #
class CapacityPolicy:
    """Peak-plus-headroom policy.  For each expert: peak = max count over the last `window`
    iterations; grow at once to ceil((1+headroom)*peak) when C_e < peak (drops occurred);
    shrink to that target only when the window is full and mean count / C_e <
    shrink_util; alpha_e = C_e * n / (T_g * k) is clamped to [min_alpha, max_alpha] and C_e
    recomputed from the clamped alpha with Eq. 4.  update() returns the new capacity list,
    or None when no expert changes (no recompile)."""

    def __init__(self, n, tokens_global, k, capacities, window=20, headroom=0.15,
                 shrink_util=0.5, min_alpha=0.25, max_alpha=8.0):
        self.n, self.Tg, self.k = n, tokens_global, k
        self.caps = list(capacities)
        self.window, self.headroom = window, headroom
        self.shrink_util, self.min_alpha, self.max_alpha = shrink_util, min_alpha, max_alpha
        self.hist = []

    def _clamp(self, c):
        alpha = c * self.n / (self.Tg * self.k)
        alpha = min(max(alpha, self.min_alpha), self.max_alpha)
        return expert_capacity(alpha, self.Tg, self.k, self.n)

    def update(self, counts):
        self.hist.append([int(c) for c in counts])
        if len(self.hist) > self.window:
            self.hist.pop(0)
        new = list(self.caps)
        for e in range(self.n):
            col = [h[e] for h in self.hist]
            peak = max(col)
            target = int(math.ceil((1.0 + self.headroom) * peak))
            if self.caps[e] < peak:
                new[e] = self._clamp(target)
            elif len(col) == self.window and (sum(col) / len(col)) / self.caps[e] < self.shrink_util:
                new[e] = self._clamp(max(target, 1))
        if new == self.caps:
            return None
        self.caps = new
        return list(new)


def caching_trigger(hit_fraction: float, epoch: int, enabled: bool, enable_at=0.96,
                    disable_below=0.90, warmup_epochs=10):
    """switch caching on at >= 96 % correctly cached samples, off below 90 %, never
    before epoch 10.  Returns the new enabled state."""
    if epoch < warmup_epochs:
        return enabled
    if not enabled and hit_fraction >= enable_at:
        return True
    if enabled and hit_fraction < disable_below:
        return False
    return enabled
