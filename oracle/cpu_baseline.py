"""Reference CPU path timed on the host cores -- TEST/BENCH INFRASTRUCTURE ONLY.

Runs the NumPy port of the reference hot path (oracle/paco_numpy.py, i.e.
matmul.py:342-397 with the 32^3 NumPy leaves of matmul.py:45-50) on a bounded
sample of a BASELINE config, process-sharded over the host cores (one process
per core, each on its own row slab: rows are independent, so this is the
reference's own arithmetic without the GIL serialisation of its threaded
mode).  Prints one JSON object.

    python -m oracle.cpu_baseline --cfg 2 --rows-per-proc 32 [--procs N]
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import time

import numpy as np

from oracle import paco_numpy as PN

INF = 2**30


def cfg_inputs(cfg: int, rows: int):
    """Seeded inputs of BASELINE config ``cfg``, A truncated to ``rows``."""
    rng = np.random.default_rng(1000 + cfg)
    if cfg == 2:
        n = 8192
        A = rng.integers(0, 2**20, (n, n), dtype=np.int32)
        A[rng.random(A.shape) < 0.10] = INF
        B = rng.integers(0, 2**20, (n, n), dtype=np.int32)
        B[rng.random(B.shape) < 0.10] = INF
        return A[:rows].copy(), B, "minplus"
    if cfg == 4:
        n = 16384
        A = rng.integers(-2**20, 2**20, (n, n), dtype=np.int32)
        B = rng.integers(-2**20, 2**20, (n, n), dtype=np.int32)
        return A[:rows].copy(), B, "maxplus"
    if cfg == 1:
        A = rng.integers(-8, 9, (384, 256), dtype=np.int32)
        B = rng.integers(-8, 9, (256, 320), dtype=np.int32)
        return A[:rows].copy(), B, "int"
    raise ValueError(f"cfg{cfg} has no CPU baseline sampler")


_G: dict = {}


def _work(args):
    lo, hi = args
    A, B, kind = _G["A"], _G["B"], _G["kind"]
    a = A[lo:hi]
    t0 = time.perf_counter()
    if kind == "minplus":
        C = np.full((hi - lo, B.shape[1]), INF, np.int32)
        PN.minplus_sat(a, B, C)
    elif kind == "maxplus":
        C = np.full((hi - lo, B.shape[1]), -INF, np.int32)
        PN.maxplus(a, B, C)
    else:
        C = np.zeros((hi - lo, B.shape[1]), np.int64)
        PN.mm_seq(a.astype(np.int64), B.astype(np.int64), C, "int")
    return time.perf_counter() - t0


def measure(cfg: int, rows_per_proc: int, procs: int | None = None, repeat: int = 1) -> dict:
    procs = procs or len(os.sched_getaffinity(0))
    A, B, kind = cfg_inputs(cfg, rows_per_proc * procs)
    _G.update(A=A, B=B, kind=kind)
    slabs = [(i * rows_per_proc, (i + 1) * rows_per_proc) for i in range(procs)]
    ctx = mp.get_context("fork")
    n_rows = rows_per_proc * procs
    ops = 2.0 * n_rows * B.shape[1] * B.shape[0]
    values, walls, per = [], [], [0.0]
    with ctx.Pool(procs) as pool:
        for _ in range(repeat):
            t0 = time.perf_counter()
            per = pool.map(_work, slabs)
            wall = time.perf_counter() - t0
            walls.append(wall)
            values.append(ops / wall / 1e9)
    wall = walls[-1]
    return {
        "value": values[-1],
        "values": values,
        "unit": "Gop/s",
        "cores": procs,
        "kind": "port",
        "wall_s": wall,
        "slowest_proc_s": max(per),
        "sample": (f"cfg{cfg}: {n_rows} of the rows of A (full k={B.shape[0]}, m={B.shape[1]}), "
                   f"{procs} processes x {rows_per_proc}-row slabs, reference mm_seq recursion "
                   f"with 32^3 NumPy leaves (oracle/paco_numpy.py)"),
    }


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def measure_threaded(cfg: int, rows: int, threads: int | None = None) -> dict:
    """The reference's shipped parallel mode on a row slab: mm_execute(
    mm_one_piece_partition(rows, m, k, P), ..., mode="parallel") with P worker
    threads (core.py:299-326; the one-piece plan is the product planner's,
    byte-identical to the reference's by tests/test_plans.py), (min,+) int64."""
    from paper_2011_01441_b200.cuboid import mm_one_piece_partition

    threads = threads or len(os.sched_getaffinity(0))
    A, B, kind = cfg_inputs(cfg, rows)
    n, k = A.shape
    m = B.shape[1]
    plan = mm_one_piece_partition(n, m, k, threads)
    if kind == "minplus":
        A64, B64 = A.astype(np.int64), B.astype(np.int64)
        C = np.full((n, m), PN.MINPLUS_INF, np.int64)
        sem = "minplus"
    elif kind == "maxplus":
        A64, B64 = -A.astype(np.int64), -B.astype(np.int64)
        C = np.full((n, m), PN.MINPLUS_INF, np.int64)
        sem = "minplus"
    else:
        A64, B64, C, sem = A.astype(np.int64), B.astype(np.int64), np.zeros((n, m), np.int64), "int"
    t0 = time.perf_counter()
    PN.mm_execute_parallel(plan, A64, B64, C, sem)
    wall = time.perf_counter() - t0
    ops = 2.0 * n * m * k
    return {"value": ops / wall / 1e9, "unit": "Gop/s", "cores": threads, "wall_s": wall,
            "sample": (f"cfg{cfg}: {n} rows of A (full k={k}, m={m}), mm_execute(mm_one_piece_partition"
                       f"({n}, {m}, {k}, {threads}), mode='parallel'): {threads} worker threads, 32^3 NumPy leaves "
                       "(oracle/paco_numpy.py mm_execute_parallel; GIL-bound like the reference's own)")}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--rows-per-proc", type=int, default=32)
    ap.add_argument("--procs", type=int, default=None)
    ap.add_argument("--repeat", type=int, default=1)
    a = ap.parse_args()
    print(json.dumps(measure(a.cfg, a.rows_per_proc, a.procs, a.repeat)))
