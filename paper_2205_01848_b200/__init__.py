"""B200-native hot path of the DynaMoE MoE layer (arXiv 2205.01848).

The compute lives in libdynamoe_b200.so (C ABI: include/moe.h, sources: csrc/).
This package is the thin Python binding (argument marshalling, workspace allocation).
"""
from ._lib import MoEError, load  # noqa: F401
from .layer import CapacityPolicy, DynaMoE, MoEFunction, MoELayer, capacity_from_factors  # noqa: F401
from .runtime import (AssignmentCache, GraphedStep, MetricQueue, RecompileRuntime,  # noqa: F401
                      caching_trigger, capacity_trigger)

__all__ = ["MoELayer", "MoEFunction", "DynaMoE", "CapacityPolicy", "capacity_from_factors",
           "MoEError", "load", "AssignmentCache", "GraphedStep", "MetricQueue", "RecompileRuntime", "caching_trigger",
           "capacity_trigger"]
