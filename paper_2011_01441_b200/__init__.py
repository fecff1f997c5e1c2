"""B200-native PACO semiring matrix multiply (arxiv 2011.01441 hot path).

Drop-in for the reference package's semiring-MM and Strassen path
(``paco.core`` + ``paco.matmul`` + the spec'd ``paco.strassen``): same plan
vocabulary and partitioners, with every arithmetic task executed by
hand-written sm_100a kernels behind the C ABI in ``include/paco_b200.h``.

As in the reference, the package root re-exports the plan/engine API
(/root/reference/pkg/src/paco/__init__.py:9-33); the MM and Strassen entry
points live in ``.matmul`` and ``.strassen``.
"""

from .engine import execute_plan
from .plan import (
    COMPUTE,
    MERGE,
    REDUCE,
    CostReport,
    Plan,
    PlanError,
    ProcList,
    Task,
    pruned_bfs_assign,
)

__all__ = [
    "COMPUTE",
    "MERGE",
    "REDUCE",
    "CostReport",
    "Plan",
    "PlanError",
    "ProcList",
    "Task",
    "execute_plan",
    "pruned_bfs_assign",
]

__version__ = "0.1.0"
