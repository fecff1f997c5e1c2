"""Import-path alias of the reference's ``paco.core`` (plan vocabulary + engine)."""

from .engine import execute_plan
from .plan import (COMPUTE, MERGE, PARALLEL, REDUCE, SERIAL_SIM, CostReport, Plan, PlanError,
                   ProcList, Task, pruned_bfs_assign, simulate_clocks)

__all__ = ["COMPUTE", "MERGE", "PARALLEL", "REDUCE", "SERIAL_SIM", "CostReport", "Plan",
           "PlanError", "ProcList", "Task", "execute_plan", "pruned_bfs_assign", "simulate_clocks"]
