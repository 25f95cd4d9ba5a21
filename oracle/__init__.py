"""fp64 CPU oracle of the DynaMoE MoE-layer hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and --impl reference)
may import this package.  The CUDA product path never imports it.  See moe_oracle.py.
"""
