"""Seeded sweep of layer shapes x routing regimes x fusion flags against the fp64 oracle
(routing bit-exact, values within the dtype budget).  Shapes are drawn to hit the kernel
variants: 1-CTA and 2-CTA tcgen05 GEMMs (BN 128 / 256), n not a multiple of 64, k up to 8,
d_out != d, ragged T (including T < one routing tile), capacity factors from heavy drops to
none, every N2 fusion flag."""
import numpy as np
import pytest

from parity_util import assert_routing_exact, assert_values, run_pair

pytestmark = pytest.mark.gpu


def _cases():
    rng = np.random.default_rng(2205)
    out = []
    for i in range(160):
        dtype = "bf16" if i % 3 else "f32"
        n = int(rng.choice([3, 8, 16, 40, 64, 130]))
        k = int(min(n, rng.choice([1, 1, 2, 2, 4, 8])))
        d = int(rng.choice([64, 128, 192, 256]))
        f = int(rng.choice([64, 128, 256, 384, 512]))
        d_out = int(rng.choice([0, 0, 128, 64]))
        T = int(rng.choice([1, 5, 127, 300, 777, 1500]))
        alpha = float(rng.choice([0.25, 0.5, 1.0, 1.25, 2.0, 7.0]))
        renorm = int(rng.integers(0, 2))
        regime = str(rng.choice(["uniform", "skewed", "ties"]))
        fusion = int(rng.choice([0, 2, 4, 6, 7]))
        out.append((dtype, n, k, d, f, d_out, T, alpha, renorm, regime, fusion))
    return out


@pytest.mark.parametrize("dtype,n,k,d,f,d_out,T,alpha,renorm,regime,fusion", _cases())
def test_fuzz_vs_oracle(dtype, n, k, d, f, d_out, T, alpha, renorm, regime, fusion):
    from paper_2205_01848_b200 import MoELayer, capacity_from_factors
    caps = capacity_from_factors([alpha] * n, T, k)
    layer = MoELayer(n, k, d, f, d_out, T, dtype, renorm, device="cuda")
    layer.set_fusion(fusion)
    layer, gpu, st, gr, own = run_pair(n, k, d, f, T, dtype, caps, renorm=renorm, regime=regime,
                                       d_out=d_out or None, layer=layer)
    assert_routing_exact(gpu, st, k)
    assert_values(gpu, st, gr, own, dtype)


def _ep_cases():
    rng = np.random.default_rng(1848)
    out = []
    for i in range(30):
        R = int(rng.choice([2, 4]))
        n = R * int(rng.choice([1, 2, 4, 8]))
        k = int(min(n, rng.choice([1, 2, 2, 4])))
        dtype = "f32" if i % 4 == 0 else "bf16"
        d = int(rng.choice([64, 128, 192]))
        f = int(rng.choice([64, 128, 256]))
        T = int(rng.choice([64, 200, 512]))
        renorm = int(rng.integers(0, 2))
        transport = str(rng.choice(["peer", "nccl"]))
        out.append((R, n, k, dtype, d, f, T, renorm, transport))
    return out


@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("R,n,k,dtype,d,f,T,renorm,transport", _ep_cases())
def test_fuzz_ep_virtual_ranks(R, n, k, dtype, d, f, T, renorm, transport):
    """R expert-parallel ranks (threads on one GPU; peer windows or the virtual communicator)
    against the single-GPU layer on the concatenated batch: routing, y, dx and each owner's
    expert gradients bitwise equal (dW_g within tolerance: summed in another split)."""
    from test_gpu_ep import _check_virtual, _run_virtual
    out, ref = _run_virtual(R, n, k, T, d, f, dtype, renorm, transport=transport)
    _check_virtual(out, ref, R, n, dtype)
