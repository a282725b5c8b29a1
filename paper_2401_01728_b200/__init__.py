"""B200-native Parallel Multi-Ring All-Reduce for Ravnest (arXiv 2401.01728).

Public surface mirrors the reference's averaging API
(/root/reference/pkg/src/ravnest/__init__.py:29-34 and multiring.py):
``RingSchedule``, ``build_ring_schedule``, ``validate_schedule``,
``chunk_bounds``, ``allreduce_cost``, ``run_allreduce``, ``apply_ring_mean``,
``AllReduceController``.  The compute path is libravnest_b200.so (sm_100a
CUDA, C ABI in include/ravnest_b200.h); importing this package does not need
a GPU, calling the averaging functions does.
"""

from .errors import ConfigError, LayoutError, ProtocolError, RavnestError, SchemaError, StallError
from .schedule import (
    CostReport,
    ParamRange,
    Ring,
    RingCost,
    RingSchedule,
    RingStats,
    allreduce_cost,
    build_ring_schedule,
    bytes_per_member,
    chunk_bounds,
    validate_schedule,
)
from .multiring import AllReduceController, apply_ring_mean, default_node_name, ring_mean_, run_allreduce

__version__ = "0.1.0"

__all__ = [
    "AllReduceController",
    "ConfigError",
    "CostReport",
    "LayoutError",
    "ParamRange",
    "ProtocolError",
    "RavnestError",
    "SchemaError",
    "Ring",
    "RingCost",
    "RingSchedule",
    "RingStats",
    "StallError",
    "allreduce_cost",
    "apply_ring_mean",
    "build_ring_schedule",
    "bytes_per_member",
    "chunk_bounds",
    "default_node_name",
    "ring_mean_",
    "run_allreduce",
    "validate_schedule",
]
