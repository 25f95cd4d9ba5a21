"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the MoE method (no gating, routing, expert or
combine math).  It only draws random tensors with the shapes and value
distributions of the paper's workloads (SURVEY.md §8(d) "Synthetic inputs") and
names the BASELINE.json configurations.  Both the oracle (oracle/) and the CUDA
path (paper_2205_01848_b200/) consume its outputs; neither is imported here.
"""
from .configs import CONFIGS, MoEShape, get_config  # noqa: F401
from .inputs import (  # noqa: F401
    make_layer,
    make_dy,
    perturb_cached,
    to_numpy64,
)
