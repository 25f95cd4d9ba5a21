"""Per-sample assignment cache (N4; S4.2 P:245-256, SPEC cache_step / cached_route S:252-267)
on the GPU against the oracle's AssignmentCache: several "epochs" over a sample set with a
drifting gate, caching switched from observe to cached routing, new samples falling back."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from parity_util import TOL, rel
from synth import make_dy, make_layer, to_numpy64

pytestmark = pytest.mark.gpu


def _layer(n, k, d, f, T, dtype, renorm=1):
    from paper_2205_01848_b200 import MoELayer
    return MoELayer(n, k, d, f, 0, T, dtype, renorm, device="cuda")


@pytest.mark.parametrize("dtype,k,renorm,d", [("bf16", 2, 1, 64), ("f32", 1, 0, 64),
                                              ("bf16", 1, 0, 64), ("bf16", 1, 0, 128)])
def test_cache_epochs_match_oracle(dtype, k, renorm, d):
    """d = 128: 2-CTA GEMMs, the histogram inside the gate epilogue (modes 0 / 3), the fused
    combine (uncached modes) and dispatch backward."""
    from paper_2205_01848_b200 import AssignmentCache
    n, f, T, N = 16, 2 * d, 256, 768
    rng = np.random.default_rng(3)
    cpu = make_layer(n, d, f, d, N, dtype)
    g = {kk: v.cuda() for kk, v in cpu.items()}
    X = g["x"]                                   # the sample set: row s = sample s
    caps = O.capacities_from_factors([1.25] * n, T, k)
    layer = _layer(n, k, d, f, T, dtype, renorm)
    layer.set_capacities(caps)
    cache = AssignmentCache(layer, N)
    ref = O.AssignmentCache(N, k)
    modes = []
    wg = g["w_gate"].clone()
    for epoch in range(4):
        if epoch == 2:
            cache.enabled = True                 # the trigger switched caching on
        # the gate drifts a little between epochs: some assignments change
        wg = (wg.float() + 0.02 * torch.randn_like(wg.float())).to(wg.dtype)
        perm = rng.permutation(N)
        for b in range(N // T - (1 if epoch == 3 else 0)):
            ids = perm[b * T:(b + 1) * T]
            if epoch == 3 and b == 0:            # 16 never-seen samples in this batch
                new = ids[rng.choice(T, 16, replace=False)]
                cache.seen[new] = False
                ref.table[new] = -1
                cache.table[torch.from_numpy(new).cuda()] = -1
            mode = cache.bind(ids)
            modes.append(mode)
            xb = X[torch.from_numpy(ids).cuda()].contiguous()
            y = layer.forward(xb, wg, g["w1"], g["b1"], g["w2"], g["b2"])
            assert layer.check_flags() == (0, 0)
            rt = layer.routing(T)
            st = layer.stats()
            logits = rt["logits"].cpu().numpy().astype(np.float64)
            fresh = O.topk_sorted(logits, k)
            assert np.array_equal(rt["fresh_idx"].cpu().numpy(), fresh)
            p64 = {kk: to_numpy64(v) for kk, v in cpu.items() if kk != "x"}
            p64["w_gate"] = to_numpy64(wg)
            want_hits = int(round(ref.hit_fraction(ids, fresh) * T))
            assert st["hit_count"] == want_hits, (epoch, b, mode)
            if mode in (1, 2):
                rows = ref.table[ids].copy()
                o = O.moe_forward(to_numpy64(xb), p64, k, caps, renorm, cached_idx=rows,
                                  logits=logits, emulate_bf16=(dtype == "bf16"),
                                  cache_fallback=(mode == 2))
            else:
                o = O.moe_forward(to_numpy64(xb), p64, k, caps, renorm, logits=logits,
                                  emulate_bf16=(dtype == "bf16"))
            assert np.array_equal(rt["idx"].cpu().numpy(), o.idx), (epoch, b, mode)
            assert np.array_equal(rt["slot_of"].cpu().numpy(), o.routing.slot_of)
            assert rel(to_numpy64(y), o.y) <= TOL[dtype]
            ref.update(ids, fresh)
            # cache_step: the device table holds this batch's fresh decisions
            assert np.array_equal(cache.table[torch.from_numpy(ids).cuda()].cpu().numpy(), fresh)
            gr = layer.backward(make_dy(T, d, dtype).cuda())
            assert torch.isfinite(gr["dx"].float()).all()
    assert 3 in modes and 1 in modes and 2 in modes


def test_cache_all_known_contract_violation_flags():
    """mode 1 promises every sample is known: a -1 row raises device flag 2, no crash."""
    n, k, d, f, T = 8, 2, 64, 128, 128
    cpu = make_layer(n, d, f, d, T, "bf16")
    g = {kk: v.cuda() for kk, v in cpu.items()}
    layer = _layer(n, k, d, f, T, "bf16")
    table = torch.full((T, k), -1, dtype=torch.int32, device="cuda")
    table[1:] = torch.tensor([0, 1], dtype=torch.int32, device="cuda")
    ids = torch.arange(T, dtype=torch.int64, device="cuda")
    layer.set_assignment_cache(table, ids, 1)
    layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    rt = layer.routing(T)
    assert layer.check_flags() == (7, 2)          # MOE_ERR_DEVICE_FLAG, invalid cached index
    assert (rt["slot_of"][0] == -1).all()          # the invalid row's pairs were dropped
    # out-of-range sample id -> flag 4
    layer.backward(make_dy(T, d, "bf16").cuda())
    bad = ids.clone()
    bad[5] = 10 ** 6
    layer.set_assignment_cache(table, bad, 2)
    layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    assert layer.check_flags() == (7, 4)          # sample id out of range
    layer.set_assignment_cache(None, None, 0)
