"""Strassen split_leftover execution check (dev tool): p dtype mode repeats."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2011_01441_b200 import strassen as S
from paper_2011_01441_b200.strassen import LeafPiece, LeafFold
p = int(sys.argv[1]); dt = sys.argv[2]
rng = np.random.default_rng(10 + p)
n = 512
A = rng.integers(-30, 30, (n, n)).astype(np.int64); B = rng.integers(-30, 30, (n, n)).astype(np.int64)
if dt == "f32":
    A = A.astype(np.float32); B = B.astype(np.float32)
plan = S.strassen_paco_partition(n, p, base=64, split_leftover=not os.environ.get("NOSPLIT"))
if os.environ.get("VERBOSE"):
    for t in plan.tasks:
        if isinstance(t.region, (LeafPiece, LeafFold)):
            print(t.id, t.kind, t.workers(), t.deps, t.region)
mode = sys.argv[3] if len(sys.argv) > 3 else "serial_sim"
for _ in range(int(sys.argv[4]) if len(sys.argv) > 4 else 1):
    C = S.strassen_execute(plan, A, B, mode)
err = np.abs(C - A.astype(np.float64) @ B)
print("ok", err.max())
if err.max() > 0:
    r, c = np.nonzero(err > 0)
    print("wrong:", len(r), "rows", r.min(), r.max(), "cols", c.min(), c.max())
    bad = sorted({(i // 64, j // 64) for i, j in zip(r, c)})
    print("64-blocks:", bad[:20])
    sub = err[r.min():r.max() + 1, c.min():c.max() + 1] > 0
    print("pattern rows:", np.nonzero(sub.any(1))[0][:40] + r.min())
    print("pattern cols:", np.nonzero(sub.any(0))[0][:70] + c.min())
