"""NumPy restatement of the reference's CPU hot path -- TEST INFRASTRUCTURE ONLY.

This is the reference algorithm as the reference runs it (the "port" kind of
CPU baseline in bench.py, and a second oracle for tests):

* ``block_int`` / ``block_minplus``  -- matmul.py:45-50 (32^3 NumPy leaves)
* ``mm_seq`` / ``_rec``               -- matmul.py:342-397 (halve the longest
  axis, ties n -> m -> k, until max extent <= base)
* ``mm_execute_serial``               -- matmul.py:417-462 in serial order:
  temps filled with zero, COMPUTE -> mm_seq into C or a temp view, REDUCE ->
  copyto(t, vadd(t, temp)) then temp.fill(zero)
* ``mm_execute_parallel``             -- the same runner from one host thread
  per worker, each task after its dependencies (core.py:299-326: a REDUCE
  runs on its first worker's thread), i.e. the reference's shipped
  ``mode="parallel"``
* ``strassen``                        -- the spec'd (absent) strassen_seq,
  SPEC.md:490-498 + PAPER.md:1839-1852, float64 or int64 ring, fixed levels

Plans are consumed duck-typed (tasks with kind/region/worker, meta dict), so
plans from either the reference or the product planner work.
"""

from __future__ import annotations

import numpy as np

MINPLUS_INF = np.int64(2**62)


def block_int(C, A, B):
    C += A @ B


def block_minplus(C, A, B):
    np.minimum(C, np.min(A[:, :, None] + B[None, :, :], axis=1), out=C)


SEMIRINGS = {
    # name: (dtype, zero, block, vadd)
    "int": (np.int64, np.int64(0), block_int, lambda x, y: x + y),
    "f64": (np.float64, 0.0, block_int, lambda x, y: x + y),
    "minplus": (np.int64, MINPLUS_INF, block_minplus, np.minimum),
}


def _axis(n, m, k):
    if n >= m and n >= k:
        return "n"
    return "m" if m >= k else "k"


def _rec(A, B, C, i0, j0, l0, n, m, k, block, base):
    if max(n, m, k) <= base:
        block(C[i0:i0 + n, j0:j0 + m], A[i0:i0 + n, l0:l0 + k], B[l0:l0 + k, j0:j0 + m])
        return
    ax = _axis(n, m, k)
    if ax == "n":
        h = n // 2
        _rec(A, B, C, i0, j0, l0, h, m, k, block, base)
        _rec(A, B, C, i0 + h, j0, l0, n - h, m, k, block, base)
    elif ax == "m":
        h = m // 2
        _rec(A, B, C, i0, j0, l0, n, h, k, block, base)
        _rec(A, B, C, i0, j0 + h, l0, n, m - h, k, block, base)
    else:
        h = k // 2
        _rec(A, B, C, i0, j0, l0, n, m, h, block, base)
        _rec(A, B, C, i0, j0, l0 + h, n, m, k - h, block, base)


def mm_seq(A, B, C, semiring: str = "int", base: int = 32) -> None:
    n, k = A.shape
    k2, m = B.shape
    if k != k2 or C.shape != (n, m):
        raise ValueError(f"shape mismatch: A{A.shape} B{B.shape} C{C.shape}")
    _rec(A, B, C, 0, 0, 0, n, m, k, SEMIRINGS[semiring][2], base)


def mm_execute_serial(plan, A, B, C, semiring: str = "int") -> None:
    dtype, zero, block, vadd = SEMIRINGS[semiring]
    reduces = plan.meta["reduces"]
    shapes = {spec[0]: (spec[4], spec[5]) for spec in reduces.values()}
    temps = {bid: np.full(shapes[bid], zero, dtype=dtype) for bid in plan.meta["temp_sizes"]}
    base = plan.meta.get("base") or 32
    for t in plan.tasks:
        if t.kind == "compute":
            c = t.region
            out = C if c.out == 0 else temps[c.out]
            mm_seq(A[c.i0:c.i0 + c.n, c.l0:c.l0 + c.k], B[c.l0:c.l0 + c.k, c.j0:c.j0 + c.m],
                   out[c.out_i0:c.out_i0 + c.n, c.out_j0:c.out_j0 + c.m], semiring, base)
        elif t.kind == "reduce":
            bid, tgt, oi, oj, n, m = reduces[t.id]
            target = C if tgt == 0 else temps[tgt]
            view = target[oi:oi + n, oj:oj + m]
            np.copyto(view, vadd(view, temps[bid]))
            temps[bid].fill(zero)


def _runner(plan, A, B, C, semiring):
    dtype, zero, block, vadd = SEMIRINGS[semiring]
    reduces = plan.meta["reduces"]
    shapes = {spec[0]: (spec[4], spec[5]) for spec in reduces.values()}
    temps = {bid: np.full(shapes[bid], zero, dtype=dtype) for bid in plan.meta["temp_sizes"]}
    base = plan.meta.get("base") or 32

    def run(t):
        if t.kind == "compute":
            c = t.region
            out = C if c.out == 0 else temps[c.out]
            mm_seq(A[c.i0:c.i0 + c.n, c.l0:c.l0 + c.k], B[c.l0:c.l0 + c.k, c.j0:c.j0 + c.m],
                   out[c.out_i0:c.out_i0 + c.n, c.out_j0:c.out_j0 + c.m], semiring, base)
        elif t.kind == "reduce":
            bid, tgt, oi, oj, n, m = reduces[t.id]
            target = C if tgt == 0 else temps[tgt]
            view = target[oi:oi + n, oj:oj + m]
            np.copyto(view, vadd(view, temps[bid]))
            temps[bid].fill(zero)
    return run


def mm_execute_parallel(plan, A, B, C, semiring: str = "int") -> None:
    """core.py:299-326 restated: worker threads, dependency events, first error re-raised."""
    import threading

    run = _runner(plan, A, B, C, semiring)
    done = [threading.Event() for _ in plan.tasks]
    mine = [[t for t in plan.tasks if t.workers()[0] == w] for w in range(plan.p)]
    errors = []

    def loop(w):
        for t in mine[w]:
            for d in t.deps:
                done[d].wait()
            if not errors:
                try:
                    run(t)
                except BaseException as exc:  # noqa: BLE001 -- re-raised after the join
                    errors.append(exc)
            done[t.id].set()

    ths = [threading.Thread(target=loop, args=(w,)) for w in range(plan.p)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    if errors:
        raise errors[0]


def minplus_sat(A32, B32, C32):
    """SEMIRING_MINPLUS on int64 copies, clamped to 2^30 (cfg2's semantics)."""
    C = C32.astype(np.int64)
    mm_seq(A32.astype(np.int64), B32.astype(np.int64), C, "minplus")
    return np.minimum(C, 2**30).astype(np.int32)


def maxplus(A32, B32, C32):
    """(max,+) through the reference min-plus by negation."""
    C = (-C32.astype(np.int64))
    mm_seq(-A32.astype(np.int64), -B32.astype(np.int64), C, "minplus")
    return np.maximum(-C, -(2**30)).astype(np.int32)


# Strassen identities, 1-indexed as in PAPER.md:1839-1852:
# (coefficient, quadrant) lists for S_r (of A), T_r (of B) and the C blocks.
S_TERMS = {1: ((1, "00"), (1, "11")), 2: ((1, "10"), (1, "11")), 3: ((1, "00"),), 4: ((1, "11"),),
           5: ((1, "00"), (1, "01")), 6: ((1, "10"), (-1, "00")), 7: ((1, "01"), (-1, "11"))}
T_TERMS = {1: ((1, "00"), (1, "11")), 2: ((1, "00"),), 3: ((1, "01"), (-1, "11")),
           4: ((1, "10"), (-1, "00")), 5: ((1, "11"),), 6: ((1, "00"), (1, "01")),
           7: ((1, "10"), (1, "11"))}
C_TERMS = {"00": ((1, 1), (1, 4), (-1, 5), (1, 7)), "01": ((1, 3), (1, 5)),
           "10": ((1, 2), (1, 4)), "11": ((1, 1), (1, 3), (-1, 2), (1, 6))}


def _quad(X, q):
    h = X.shape[0] // 2
    r, c = int(q[0]), int(q[1])
    return X[r * h:(r + 1) * h, c * h:(c + 1) * h]


def _combine(X, terms):
    out = None
    for coef, q in terms:
        part = _quad(X, q)
        out = part.copy() if out is None and coef > 0 else (
            -part if out is None else (out + part if coef > 0 else out - part))
    return out


def strassen(A, B, levels: int, leaf=None):
    """C = A x B with ``levels`` Strassen levels over the ring of A's dtype.

    n must be divisible by 2**levels; leaves use ``leaf`` (default A @ B).
    """
    n = A.shape[0]
    if levels == 0 or n == 1 or n % 2:
        return leaf(A, B) if leaf else A @ B
    M = {r: strassen(_combine(A, S_TERMS[r]), _combine(B, T_TERMS[r]), levels - 1, leaf)
         for r in range(1, 8)}
    C = np.empty((n, n), dtype=np.result_type(A, B))
    h = n // 2
    for q, terms in C_TERMS.items():
        acc = None
        for coef, r in terms:
            acc = (M[r].copy() if coef > 0 else -M[r]) if acc is None else (
                acc + M[r] if coef > 0 else acc - M[r])
        r0, c0 = int(q[0]) * h, int(q[1]) * h
        C[r0:r0 + h, c0:c0 + h] = acc
    return C
