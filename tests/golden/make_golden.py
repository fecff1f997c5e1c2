"""Generate the golden fixtures by running the REFERENCE itself (this container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed, small):
  plans.json.gz  -- reference Plan.dump_text() + meta for a grid of shapes, p and
                    variants (mm_paco_partition / mm_one_piece_partition /
                    mm_hetero_partition, matmul.py:214-339)
  mm_cases.npz   -- seeded operands and the reference's mm_execute results
                    (matmul.py:417-462) for every semiring the hot path covers,
                    including cfg1 at full size.

Seeds follow SURVEY.md 8(d): numpy default_rng(1000 + cfg#), A drawn before B.
The generated files are read by tests/ on any machine; /root/reference is not
needed at test time.
"""

from __future__ import annotations

import gzip
import json
import os
import random

import numpy as np
import paco.matmul as R  # the reference package (PYTHONPATH=/root/reference/pkg/src)

HERE = os.path.dirname(os.path.abspath(__file__))


def plan_record(kind, args, plan):
    meta = dict(plan.meta)
    meta["temp_sizes"] = {str(k): v for k, v in meta["temp_sizes"].items()}
    meta["reduces"] = {str(k): list(v) for k, v in meta["reduces"].items()}
    return {"kind": kind, "args": list(args), "dump": plan.dump_text(), "meta": meta}


def make_plans():
    rnd = random.Random(2011_01441)
    shapes = [(384, 320, 256), (8192, 8192, 8192), (16384, 16384, 16384), (65536, 1024, 256),
              (8, 4, 2), (9, 4, 2), (32, 32, 32), (64, 64, 64), (17, 9, 5), (1, 1, 1), (3, 100, 7),
              (4096, 4096, 4096), (128, 128, 128), (512, 512, 512)]
    shapes += [tuple(rnd.randint(1, 160) for _ in range(3)) for _ in range(60)]
    out = []
    for s in shapes:
        for p in (1, 2, 3, 4, 5, 6, 7, 8, 13, 148):
            for kind in ("one_piece", "paco"):
                if kind == "paco" and (max(s) > 4096 and p > 8 or max(s) >= 16384):
                    continue
                fn = R.mm_one_piece_partition if kind == "one_piece" else R.mm_paco_partition
                try:
                    plan = fn(*s, p)
                except R.PlanError as e:
                    out.append({"kind": kind, "args": [*s, p], "error": str(e)})
                    continue
                out.append(plan_record(kind, (*s, p), plan))
        for w in ((1.0,), (3.0, 1.0), (1.0, 1.0), (3.0, 1.0, 1.0, 1.0), (1.5, 2.5, 1.0),
                  (1.0, 1.02, 0.97, 1.0, 1.01, 0.99, 1.0, 1.03)):
            try:
                plan = R.mm_hetero_partition(*s, w)
            except R.PlanError as e:
                out.append({"kind": "hetero", "args": [*s, list(w)], "error": str(e)})
                continue
            out.append(plan_record("hetero", (*s, list(w)), plan))
    with gzip.open(os.path.join(HERE, "plans.json.gz"), "wt") as f:
        json.dump(out, f)
    return len(out)


def run(plan, A, B, C, sr):
    R.mm_execute(plan, A, B, C, sr)
    return C


def make_mm_cases():
    cases = {}

    # cfg1, full size: (+,x) int32 [-8,8] -> int64, PACO p=3 (BASELINE.json configs[0])
    rng = np.random.default_rng(1001)
    A = rng.integers(-8, 9, (384, 256), dtype=np.int32)
    B = rng.integers(-8, 9, (256, 320), dtype=np.int32)
    C = run(R.mm_paco_partition(384, 320, 256, 3), A.astype(np.int64), B.astype(np.int64),
            np.zeros((384, 320), np.int64), R.SEMIRING_INT)
    assert np.array_equal(C, R.mm_oracle(A.astype(np.int64), B.astype(np.int64), R.SEMIRING_INT))
    cases.update(cfg1_A=A, cfg1_B=B, cfg1_C=C)

    # cfg2 distribution, reduced size: (min,+) int32 [0,2^20) with 10% INF=2^30
    rng = np.random.default_rng(1002)
    n, m, k = 96, 80, 112
    A = rng.integers(0, 2**20, (n, k), dtype=np.int32)
    A[rng.random(A.shape) < 0.10] = 2**30
    B = rng.integers(0, 2**20, (k, m), dtype=np.int32)
    B[rng.random(B.shape) < 0.10] = 2**30
    C64 = run(R.mm_one_piece_partition(n, m, k, 5), A.astype(np.int64), B.astype(np.int64),
              np.full((n, m), R.MINPLUS_INF, np.int64), R.SEMIRING_MINPLUS)
    cases.update(minplus_sat_A=A, minplus_sat_B=B,
                 minplus_sat_C=np.minimum(C64, 2**30).astype(np.int32))

    # all-INF rows/cols edge case for the saturating semiring
    A2 = A.copy()
    A2[:7] = 2**30
    B2 = B.copy()
    B2[:, -5:] = 2**30
    C64 = run(R.mm_one_piece_partition(n, m, k, 3), A2.astype(np.int64), B2.astype(np.int64),
              np.full((n, m), R.MINPLUS_INF, np.int64), R.SEMIRING_MINPLUS)
    cases.update(minplus_inf_A=A2, minplus_inf_B=B2,
                 minplus_inf_C=np.minimum(C64, 2**30).astype(np.int32))

    # cfg4 distribution, reduced size: (max,+) via the reference min-plus on negated inputs
    rng = np.random.default_rng(1004)
    n, m, k = 80, 72, 100
    A = rng.integers(-2**20, 2**20, (n, k), dtype=np.int32)
    B = rng.integers(-2**20, 2**20, (k, m), dtype=np.int32)
    negC = run(R.mm_one_piece_partition(n, m, k, 7), -A.astype(np.int64), -B.astype(np.int64),
               np.full((n, m), R.MINPLUS_INF, np.int64), R.SEMIRING_MINPLUS)
    cases.update(maxplus_A=A, maxplus_B=B, maxplus_C=(-negC).astype(np.int32))

    # the reference (min,+) verbatim: int64, INF 2^62, wrapping INF+INF (matmul.py:29,49-50)
    rng = np.random.default_rng(7)
    n, m, k = 40, 36, 44
    A = rng.integers(-2**40, 2**40, (n, k), dtype=np.int64)
    A[rng.random(A.shape) < 0.3] = R.MINPLUS_INF
    B = rng.integers(-2**40, 2**40, (k, m), dtype=np.int64)
    B[rng.random(B.shape) < 0.3] = R.MINPLUS_INF
    with np.errstate(over="ignore"):
        C = run(R.mm_paco_partition(n, m, k, 3), A, B, np.full((n, m), R.MINPLUS_INF, np.int64),
                R.SEMIRING_MINPLUS)
    cases.update(minplus_i64_A=A, minplus_i64_B=B, minplus_i64_C=C)

    # int64 ring with wrapping products (NumPy int64 semantics)
    rng = np.random.default_rng(8)
    n, m, k = 48, 40, 52
    A = rng.integers(-2**40, 2**40, (n, k), dtype=np.int64)
    B = rng.integers(-2**40, 2**40, (k, m), dtype=np.int64)
    C0 = rng.integers(-2**60, 2**60, (n, m), dtype=np.int64)
    C = run(R.mm_one_piece_partition(n, m, k, 5), A, B, C0.copy(), R.SEMIRING_INT)
    cases.update(int_wrap_A=A, int_wrap_B=B, int_wrap_C0=C0, int_wrap_C=C)

    # float64 (+,x); C accumulates into a nonzero start
    rng = np.random.default_rng(9)
    n, m, k = 50, 45, 60
    A = rng.standard_normal((n, k))
    B = rng.standard_normal((k, m))
    C0 = rng.standard_normal((n, m))
    C = run(R.mm_one_piece_partition(n, m, k, 3), A, B, C0.copy(), R.SEMIRING_F64)
    cases.update(f64_A=A, f64_B=B, f64_C0=C0, f64_C=C)

    # cfg3 distribution, reduced size: bf16-representable operands, f64 reference result
    rng = np.random.default_rng(1003)
    n, m, k = 256, 192, 128
    A = rng.standard_normal((n, k), dtype=np.float32)
    B = rng.standard_normal((k, m), dtype=np.float32)
    # round to bf16 (RNE) in NumPy so the fixture carries the exact operand bits
    def to_bf16(x):
        b = x.view(np.uint32).astype(np.uint64)
        b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
        return (b << 16).astype(np.uint32).view(np.float32)
    A, B = to_bf16(A), to_bf16(B)
    C = run(R.mm_one_piece_partition(n, m, k, 1), A.astype(np.float64), B.astype(np.float64),
            np.zeros((n, m)), R.SEMIRING_F64)
    cases.update(bf16_A=A, bf16_B=B, bf16_C=C)

    np.savez_compressed(os.path.join(HERE, "mm_cases.npz"), **cases)
    return sorted(cases)


if __name__ == "__main__":
    print("plans:", make_plans())
    print("cases:", make_mm_cases())
