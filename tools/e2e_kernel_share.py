"""cfg2 end to end (NumPy mm_seq): sum of the library's kernel times inside one
call vs the call's wall time, per launch (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import matmul as M

INF = 2 ** 30
rng = np.random.default_rng(1002)
n = 8192
A = rng.integers(0, 2**20, (n, n), dtype=np.int32)
B = rng.integers(0, 2**20, (n, n), dtype=np.int32)
C = np.full((n, n), INF, np.int32)
for _ in range(3):
    M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
torch.cuda.synchronize()
with nat.kernel_timing() as kt:
    C.fill(INF)
    t0 = time.perf_counter()
    M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
    wall = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    fams = {f: kt.read(f) for f in range(5)}
print("wall ms", round(wall, 3))
print("kernel families (ms, launches):", {f: (round(v[0], 3), v[1]) for f, v in fams.items()})
