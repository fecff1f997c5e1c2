"""Stress the k-phased host pipeline (NumPy host, overwrite, (min,+) sat) and
report mismatches against the oracle (race hunting)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import cref
from paper_2011_01441_b200 import matmul as M

INF = 2**30
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(43)
n, m, k = 1100, 650, 2600


def trop(shape, lo, hi, f):
    x = rng.integers(lo, hi, shape, dtype=np.int32)
    x[rng.random(shape) < f] = INF
    return x


A = trop((n, k), 0, 2**20, 0.1)
B = trop((k, m), 0, 2**20, 0.1)
C0 = np.full((n, m), INF, np.int32)
want = cref.mm(cref.SR_MINPLUS_SAT32, A, B, C0.copy())
bad = 0
for r in range(reps):
    for overwrite in (True, False):
        C = np.full((n, m), 7, np.int32) if overwrite else C0.copy()
        M.mm_seq(A.copy(), B.copy(), C, M.SEMIRING_MINPLUS_SAT, overwrite=overwrite)
        if not np.array_equal(C, want):
            bad += 1
            idx = np.argwhere(C != want)
            print(f"rep {r} overwrite={overwrite}: {len(idx)} mismatches; rows {np.unique(idx[:, 0])[:20]} "
                  f"cols {np.unique(idx[:, 1])[:20]}; first {idx[:3].tolist()} got {C[tuple(idx[0])]} "
                  f"want {want[tuple(idx[0])]}", flush=True)
print("bad", bad, "of", 2 * reps)
