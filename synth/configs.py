"""BASELINE.json configurations as plain shape records (SURVEY.md §8 "Config shapes").

Values not stated in BASELINE.json are the SURVEY's proposals (marked there):
c2 d_ff = 4*d, fp32; c4 strong scaling (262,144 global tokens); c5 weak scaling
(65,536 tokens per rank).
"""
from dataclasses import dataclass, replace


@dataclass(frozen=True)
class MoEShape:
    name: str
    n_experts: int
    top_k: int
    d_model: int
    d_ff: int
    d_out: int
    tokens: int            # tokens per rank (T)
    dtype: str             # "f32" | "bf16"
    alpha: float = 1.0     # static capacity factor (Eq. 4)
    renormalize: int = 1   # 1 = Alg. 1 normalize; 0 = raw softmax prob (Switch)
    scaling: str = "strong"

    def with_(self, **kw):
        return replace(self, **kw)


CONFIGS = {
    # BASELINE.json configs[0]: single MoE layer, 4 MLP experts, top-2, d=64, f=128, 512 tokens, alpha 1.0, fp32
    "c1": MoEShape("c1", 4, 2, 64, 128, 64, 512, "f32", 1.0, 1),
    # configs[1]: MNIST/CIFAR-shaped classifier: 16 experts, top-1, d=256, batch 4096, dynamic capacity
    "c2": MoEShape("c2", 16, 1, 256, 1024, 256, 4096, "f32", 1.0, 0),
    # configs[2]: Switch-style FFN MoE: 64 experts, top-1, d=1024, f=4096, 64K tokens, bf16, 1 GPU
    "c3": MoEShape("c3", 64, 1, 1024, 4096, 1024, 65536, "bf16", 1.0, 0),
    # configs[3]: expert-parallel: 128 experts over 8 GPUs, top-2, d=2048, f=8192, 256K tokens (global)
    "c4": MoEShape("c4", 128, 2, 2048, 8192, 2048, 262144, "bf16", 1.0, 1),
    # configs[4]: caching mode, 64 experts, cached top-1 indices, dynamic capacities, 64K tokens per rank
    "c5": MoEShape("c5", 64, 1, 1024, 4096, 1024, 65536, "bf16", 1.0, 0, "weak"),
}


def get_config(name: str) -> MoEShape:
    if name not in CONFIGS:
        raise KeyError(f"unknown config {name!r}; known: {sorted(CONFIGS)}")
    return CONFIGS[name]
