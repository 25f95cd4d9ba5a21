"""Seeded synthetic tensors shaped like the paper's workloads.

Recipe (also stated in DESIGN.md §"Input recipe"):

* uniform regime: x ~ N(0,1); W_g ~ N(0, 1/d) so logits are about N(0,1);
  W1 ~ N(0, 1/d); W2 ~ N(0, 1/f); b1, b2 ~ N(0, 0.1^2); dy ~ N(0,1).
* skewed regime: SPEC's clustered Gaussian: n cluster centres mu_c ~ N(0,1)^d,
  cluster popularity p_c proportional to (c+1)^-zipf_s, x = mu_c + 0.5*eps, and gate rows
  aligned with the centres, W_g[e] = 4*mu_e/d (so the home expert's logit is about 4).
  zipf_s = 0.5 gives max_e cnt_e / mean about 2-7 at n = 16..128, the imbalance
  that forced alpha = 7.0 in P:308.
* ties regime: x and W_g drawn from {-1, 0, 1}, so every fp32 logit is a small exact
  integer and top-k ties are everywhere (tie rule: lower expert index, reading 3).

Seeds (recorded by bench.py): data 1848, gate 2205, experts 1, upstream grad 7.
Values are generated in fp32 with torch's generator on the requested device and
then cast to the layer dtype; the cast (round-to-nearest-even to bf16) is input
generation, not method arithmetic.  Nothing here gates, routes or combines.
"""
from __future__ import annotations

import numpy as np
import torch

SEED_DATA = 1848
SEED_GATE = 2205
SEED_EXPERTS = 1
SEED_DY = 7

_DT = {"f32": torch.float32, "bf16": torch.bfloat16}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def make_layer(n: int, d: int, f: int, d_out: int, T: int, dtype: str = "f32",
               regime: str = "uniform", device="cpu", zipf_s: float = 0.5,
               seed_offset: int = 0):
    """Return dict x, w_gate, w1, b1, w2, b2 (torch tensors, layer dtype, on `device`).

    Layouts are torch Linear ([out, in]): w_gate [n,d], w1 [n,f,d], b1 [n,f],
    w2 [n,d_out,f], b2 [n,d_out]; x is [T,d] row-major.
    """
    dev = torch.device(device)
    dt = _DT[dtype]
    gd = _gen(SEED_DATA + seed_offset, dev)
    gg = _gen(SEED_GATE + seed_offset, dev)
    ge = _gen(SEED_EXPERTS + seed_offset, dev)
    f32 = torch.float32
    if regime == "uniform":
        x = torch.randn(T, d, generator=gd, device=dev, dtype=f32)
        wg = torch.randn(n, d, generator=gg, device=dev, dtype=f32) * (1.0 / d) ** 0.5
    elif regime == "skewed":
        mu = torch.randn(n, d, generator=gg, device=dev, dtype=f32)
        pop = torch.arange(1, n + 1, device=dev, dtype=torch.float64) ** (-zipf_s)
        pop = pop / pop.sum()
        c = torch.multinomial(pop.to(f32), T, replacement=True, generator=gd)
        x = mu[c] + 0.5 * torch.randn(T, d, generator=gd, device=dev, dtype=f32)
        wg = 4.0 * mu / d
    elif regime == "ties":
        x = torch.randint(-1, 2, (T, d), generator=gd, device=dev).to(f32)
        wg = torch.randint(-1, 2, (n, d), generator=gg, device=dev).to(f32)
    else:
        raise ValueError(f"unknown regime {regime!r}")
    w1 = torch.randn(n, f, d, generator=ge, device=dev, dtype=f32) * (1.0 / d) ** 0.5
    b1 = torch.randn(n, f, generator=ge, device=dev, dtype=f32) * 0.1
    w2 = torch.randn(n, d_out, f, generator=ge, device=dev, dtype=f32) * (1.0 / f) ** 0.5
    b2 = torch.randn(n, d_out, generator=ge, device=dev, dtype=f32) * 0.1
    out = dict(x=x, w_gate=wg, w1=w1, b1=b1, w2=w2, b2=b2)
    return {k: v.to(dt).contiguous() for k, v in out.items()}


def make_dy(T: int, d_out: int, dtype: str = "f32", device="cpu", seed_offset: int = 0):
    g = _gen(SEED_DY + seed_offset, torch.device(device))
    return torch.randn(T, d_out, generator=g, device=device, dtype=torch.float32).to(_DT[dtype])


def perturb_cached(fresh_idx: np.ndarray, n: int, miss_frac: float = 0.03, seed: int = 97):
    """Cache-converged regime: copy `fresh_idx` [T,k] and replace the rows of
    a random `miss_frac` of tokens by a random set of k distinct experts (in random order).
    `fresh_idx` is supplied by the caller (from the oracle's own top-k in tests)."""
    rng = np.random.default_rng(seed)
    T, k = fresh_idx.shape
    out = np.array(fresh_idx, dtype=np.int32, copy=True)
    miss = rng.random(T) < miss_frac
    for t in np.nonzero(miss)[0]:
        out[t] = rng.permutation(n)[:k]
    return out


def to_numpy64(t: torch.Tensor) -> np.ndarray:
    """Exact widening of a torch tensor (fp32 or bf16 values) to a float64 numpy array."""
    return t.detach().to("cpu", torch.float64).numpy()
