"""N4 recompile runtime on the GPU: the metric future queue (App. B), Delta_launch-delayed
triggers with launch-frontier effect latency, and CUDA-graph capture / re-instantiation."""
import pytest
import torch

from oracle import moe_oracle as O
from synth import make_dy, make_layer

pytestmark = pytest.mark.gpu


def _setup(n=16, k=1, T=1024, d=64, f=128, dtype="bf16", regime="skewed"):
    from paper_2205_01848_b200 import MoELayer
    g = {kk: v.cuda() for kk, v in make_layer(n, d, f, d, T, dtype, regime).items()}
    dy = make_dy(T, d, dtype).cuda()
    layer = MoELayer(n, k, d, f, 0, T, dtype, 0, device="cuda")
    return layer, g, dy


def _step(layer, g, dy):
    layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    layer.backward(dy)


def test_metric_queue_order_and_bound():
    from paper_2205_01848_b200 import MoEError
    layer, g, dy = _setup()
    q = layer.metrics_queue(3)
    for _ in range(3):
        _step(layer, g, dy)
    assert q.pending() == 3
    with pytest.raises(MoEError):            # launch frontier bounded by the queue depth
        _step(layer, g, dy)
    ref = layer.stats()
    its = [q.pop(block=True) for _ in range(3)]
    assert [m["iteration"] for m in its] == [0, 1, 2]
    assert all(m["counts"] == ref["counts"] and m["drops"] == ref["drops"] for m in its)
    assert q.pop(block=False) is None and q.pending() == 0


def test_runtime_capacity_policy_effect_latency():
    """A decision from iteration t's metrics first affects launch t + Delta + 1."""
    from paper_2205_01848_b200 import CapacityPolicy, RecompileRuntime, capacity_trigger
    n, k, T = 16, 1, 1024
    layer, g, dy = _setup(n, k, T)
    layer.set_capacity_factors([1.0] * n)
    pol = CapacityPolicy(n, T, k, layer.capacities, window=4)
    delta = 2
    rt = RecompileRuntime(layer, delta_launch=delta, triggers=[capacity_trigger(pol)])
    drops = []
    for it in range(12):
        rt.before_launch()
        _step(layer, g, dy)
        drops.append(layer.stats()["drops"])
        rt.after_launch()
    rt.drain()
    assert rt.log, "skewed routing at alpha = 1 must trigger a recompile"
    for metric_it, launched, dec in rt.log:
        assert launched == metric_it + delta + 1
    assert drops[0] > 0 and drops[-1] == 0   # dynamic capacities removed the drops


@pytest.mark.parametrize("d,f", [(64, 128), (128, 256)])
def test_graphed_step_matches_eager_and_recaptures(d, f):
    """(128, 256): every GEMM on the 2-CTA kernel with the N2 combine / dispatch-backward
    fusions and programmatic dependent launches inside the captured graph."""
    from paper_2205_01848_b200 import GraphedStep
    layer, g, dy = _setup(dtype="bf16", regime="uniform", d=d, f=f)
    layer.set_capacity_factors([1.25] * layer.n)
    layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"])
    eager = layer.backward(dy)
    y_e = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"]).clone()
    layer.backward(dy)
    torch.cuda.synchronize()
    grads = {kk: torch.empty_like(v) for kk, v in eager.items()}
    gs = GraphedStep(layer, g["x"], g, dy, grads)
    y = gs.replay().clone()
    torch.cuda.synchronize()
    assert torch.equal(y, y_e)
    for kk in eager:
        assert torch.equal(grads[kk], eager[kk]), kk
    # recompile: capacities change -> the graph is re-instantiated and matches eager again
    layer.set_capacity_factors([0.5] * layer.n)
    y2 = gs.replay().clone()
    torch.cuda.synchronize()
    y2_e = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"]).clone()
    layer.backward(dy)
    torch.cuda.synchronize()
    assert torch.equal(y2, y2_e) and not torch.equal(y2, y_e)


def test_graphed_step_recaptures_on_cached_assignment_and_fusion():
    """Setters other than capacities (cached indices, fusion flags) also change captured
    kernel arguments: the replay re-captures and matches eager; the captured cached-index
    tensor stays alive after the caller drops it."""
    import numpy as np
    from paper_2205_01848_b200 import GraphedStep
    from synth import perturb_cached
    n, k, T = 16, 1, 1024
    layer, g, dy = _setup(n, k, T, dtype="bf16", regime="uniform", d=128, f=256)
    layer.set_capacity_factors([1.25] * n)
    grads = {kk: torch.empty_like(v) for kk, v in
             dict(dx=g["x"], dw_gate=g["w_gate"], dw1=g["w1"], db1=g["b1"], dw2=g["w2"],
                  db2=g["b2"]).items()}
    gs = GraphedStep(layer, g["x"], g, dy, grads)
    y0 = gs.replay().clone()
    fresh = layer.routing(T)["fresh_idx"].cpu().numpy()
    cidx = torch.from_numpy(np.ascontiguousarray(perturb_cached(fresh, n, 0.5),
                                                 dtype=np.int32)).cuda()
    layer.set_cached_assignment(cidx)
    del cidx                                  # the graph's capture keeps it alive
    y1 = gs.replay().clone()
    y1_e = layer.forward(g["x"], g["w_gate"], g["w1"], g["b1"], g["w2"], g["b2"]).clone()
    layer.backward(dy)
    torch.cuda.synchronize()
    assert torch.equal(y1, y1_e) and not torch.equal(y1, y0)
    layer.set_cached_assignment(None)
    layer.set_fusion(0)
    y2 = gs.replay().clone()
    torch.cuda.synchronize()
    assert torch.equal(y2, y0)                # combine fusion is bitwise equal to unfused


def test_backward_of_a_stale_forward_raises():
    """One saved forward per layer: a backward after another forward (e.g. an eval pass)
    must not silently use the wrong batch (autograd path)."""
    from paper_2205_01848_b200 import DynaMoE
    torch.manual_seed(0)
    m = DynaMoE(8, 2, 64, 128, 0, 256, "f32", device="cuda")
    x = torch.randn(256, 64, device="cuda", requires_grad=True)
    y = m(x)
    with torch.no_grad():
        m(torch.randn(256, 64, device="cuda"))
    with pytest.raises(RuntimeError, match="another forward"):
        y.sum().backward()
