"""cProfile of cfg1's mm_execute call (host-side cost of the API path) (dev tool)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2011_01441_b200 import matmul as M

rng = np.random.default_rng(1001)
a = torch.from_numpy(rng.integers(-8, 9, (384, 256), dtype=np.int32)).cuda()
b = torch.from_numpy(rng.integers(-8, 9, (256, 320), dtype=np.int32)).cuda()
c = torch.zeros(384, 320, dtype=torch.int64, device="cuda")
plan = M.mm_paco_partition(384, 320, 256, 3)
for _ in range(20):
    M.mm_execute(plan, a, b, c, M.SEMIRING_INT)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    M.mm_execute(plan, a, b, c, M.SEMIRING_INT)
torch.cuda.synchronize()
print("per call ms", (time.perf_counter() - t0) / 200 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    M.mm_execute(plan, a, b, c, M.SEMIRING_INT)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
