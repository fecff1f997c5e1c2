"""Dependency-ordered plan execution (the reference engine's contract).

``execute_plan`` follows /root/reference/pkg/src/paco/core.py:245-326:
validate, compute the static cost model, then call ``runner(task)`` for every
task after its dependencies -- inline in plan order (``serial_sim``) or from
one host thread per worker (``parallel``; a task shared by several workers
runs on its first worker's thread, core.py:301-303).  The first runner
exception is re-raised after every thread has joined (core.py:304-325).

On B200 the runner only *enqueues* device work on the worker's CUDA stream and
records an event, so "dependency done" means "ordered on the device"; the
caller synchronises once at the end.  Cache simulation (``sims``, the
reference's cachesim.py) is out of scope here -- ncu counters replace it.
"""

from __future__ import annotations

import threading
from time import perf_counter
from typing import Callable

from .plan import PARALLEL, SERIAL_SIM, CostReport, Plan, PlanError, Task, simulate_clocks


def execute_plan(plan: Plan, runner: Callable[[Task], None] | None = None, mode: str = SERIAL_SIM,
                 *, sims: dict | None = None) -> CostReport:
    plan.validate()
    if mode not in (SERIAL_SIM, PARALLEL):
        raise PlanError(f"unknown mode {mode!r}")
    if sims is not None:
        raise NotImplementedError(
            "cache simulation (paco.cachesim) is out of scope on B200; profile with ncu instead")
    total, makespan = simulate_clocks(plan)
    report = CostReport(work_total=total, work_max=makespan,
                        temp_space_peak=plan.meta.get("temp_peak", 0))
    if runner is None:
        return report
    if mode == SERIAL_SIM:
        for t in plan.tasks:
            runner(t)
    else:
        report.wall_s = _threaded(plan, runner)
    return report


def _threaded(plan: Plan, runner: Callable[[Task], None]) -> float:
    finished = [threading.Event() for _ in plan.tasks]
    per_worker: list[list[Task]] = [[] for _ in range(plan.p)]
    for t in plan.tasks:
        per_worker[t.workers()[0]].append(t)
    errors: list[BaseException] = []

    def loop(w: int) -> None:
        for t in per_worker[w]:
            for d in t.deps:
                finished[d].wait()
            if not errors:
                try:
                    runner(t)
                except BaseException as exc:  # re-raised once peers are unblocked
                    errors.append(exc)
            finished[t.id].set()

    threads = [threading.Thread(target=loop, args=(w,), name=f"paco-worker-{w}")
               for w in range(plan.p)]
    start = perf_counter()
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    elapsed = perf_counter() - start
    if errors:
        raise errors[0]
    return elapsed
