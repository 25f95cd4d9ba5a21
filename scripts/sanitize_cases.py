"""Small cases for compute-sanitizer (round 2 kernels): smoke() (fp32 split-tf32 GEMMs, bf16
1- and 2-CTA GEMMs with O in token order, lean combine backward, fused combine / dispatch
backward) plus the k = 2 in-epilogue combine (MOE_FUSE_COMBINE2) and an fp32 accumulate pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import __graft_entry__ as g  # noqa: E402
from paper_2205_01848_b200 import MoELayer, capacity_from_factors  # noqa: E402
from synth import make_dy, make_layer  # noqa: E402

g.smoke()
for dtype, k, fusion in (("bf16", 2, 30), ("f32", 2, 0)):
    n, d, f, T = 8, 128, 256, 300
    w = {kk: v.cuda() for kk, v in make_layer(n, d, f, d, T, dtype).items()}
    dy = make_dy(T, d, dtype).cuda()
    layer = MoELayer(n, k, d, f, 0, T, dtype, 1, device="cuda")
    layer.set_fusion(fusion)
    layer.set_capacities(capacity_from_factors([0.8] * n, T, k))
    grads = None
    for it in range(2):
        layer.forward(w["x"], w["w_gate"], w["w1"], w["b1"], w["w2"], w["b2"])
        grads = layer.backward(dy, grads=grads, accumulate=it > 0)
    torch.cuda.synchronize()
    print("case", dtype, k, fusion, "ok", bool(torch.isfinite(grads["dw1"].float()).all()))
