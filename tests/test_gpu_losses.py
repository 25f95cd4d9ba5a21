"""N3 loss variants on the GPU vs the oracle: Eq. 3 balance term (value and its gradient
through the gate) and the AggregateSpec rows with specification-loss gradients."""
import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from parity_util import TOL, _np, checked_relu_mask, kernel_relu_mask, rel
from synth import make_dy, make_layer, to_numpy64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", [64, 128])   # 128: 2-CTA GEMMs + fused dispatch backward (k = 1)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,k,renorm", [(8, 2, 1), (16, 1, 0), (8, 2, 0)])
def test_balance_and_spec_parity(dtype, n, k, renorm, d):
    from paper_2205_01848_b200 import MoELayer
    T, f, lam = 700, 2 * d, 0.3
    caps = O.capacities_from_factors([1.0] * n, T, k)
    cpu = make_layer(n, d, f, d, T, dtype)
    dy = make_dy(T, d, dtype)
    g = torch.Generator().manual_seed(3)
    dspec = torch.randn(T * k, d, generator=g).to(cpu["x"].dtype)
    dw_ext = torch.randn(T, k, generator=g)
    layer = MoELayer(n, k, d, f, 0, T, dtype, renorm, device="cuda")
    layer.set_capacities(caps)
    layer.set_balance_loss(lam)
    layer.enable_spec(True)
    layer.set_spec_grads(dspec.cuda(), dw_ext.cuda())
    gg = {kk: v.cuda() for kk, v in cpu.items()}
    y = layer.forward(gg["x"], gg["w_gate"], gg["w1"], gg["b1"], gg["w2"], gg["b2"])
    rt = layer.routing(T)
    aux = layer.aux_loss()
    spec = _np(layer.spec[:T * k])
    valid = layer.spec_valid[:T * k].cpu().numpy()
    grads = layer.backward(dy.cuda())
    torch.cuda.synchronize()
    p64 = {kk: to_numpy64(v) for kk, v in cpu.items() if kk != "x"}
    st = O.moe_forward(to_numpy64(cpu["x"]), p64, k, caps, renorm, logits=_np(rt["logits"]).astype(np.float64),
                       emulate_bf16=(dtype == "bf16"), balance_lambda=lam)
    mask = checked_relu_mask(st, kernel_relu_mask(rt, st), "losses")
    gr = O.moe_backward(st, to_numpy64(dy), dspec=to_numpy64(dspec), dw_ext=dw_ext.double().numpy(),
                        relu_mask=mask)
    tol = TOL[dtype]
    assert abs(aux - st.extra["aux_loss"]) <= 1e-5 * abs(st.extra["aux_loss"])
    assert np.array_equal(valid, st.extra["spec_valid"])
    assert rel(spec, st.extra["spec"]) <= tol
    assert rel(to_numpy64(y), st.y) <= tol
    for key in ("dx", "dw_gate", "dw1", "db1", "dw2", "db2"):
        assert rel(to_numpy64(grads[key]), gr[key]) <= tol, key
    rt2 = layer.routing(T)
    assert rel(_np(rt2["dl"]), gr["dl"]) <= tol
    assert rel(_np(rt2["dw"]), gr["dw"]) <= tol
