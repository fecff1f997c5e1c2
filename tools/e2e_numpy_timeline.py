"""Where does the NumPy e2e of cfg2 spend its time?  Host timeline of
mm._kphased_host_mm's staging copies (thread count from argv) next to the
GPU's compute/copy events."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200 import mm as MM

threads = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8,16").split(",")]
n = 8192
rng = np.random.default_rng(1002)
A = rng.integers(0, 2**20, (n, n), dtype=np.int32)
B = rng.integers(0, 2**20, (n, n), dtype=np.int32)
C = np.full((n, n), 2**30, np.int32)
real = MM._host_copy
log = []


def traced(dst, src):
    t0 = time.perf_counter()
    real(dst, src)
    log.append((t0, time.perf_counter(), dst.nbytes))


out = {}
for T in threads:
    MM._HOST_THREADS = T
    MM._host_pool = None
    MM._host_copy = real
    M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
    ts = []
    for _ in range(3):
        C.fill(2**30)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
        ts.append((time.perf_counter() - t0) * 1e3)
    MM._host_copy = traced
    log.clear()
    C.fill(2**30)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    M.mm_seq(A, B, C, M.SEMIRING_MINPLUS_SAT)
    t1 = time.perf_counter()
    out[f"T{T}"] = {"ms": ts, "traced_ms": (t1 - t0) * 1e3,
                    "copies": [(round((a - t0) * 1e3, 2), round((b - a) * 1e3, 2), nb >> 20) for a, b, nb in log],
                    "copy_ms_total": sum(b - a for a, b, _ in log) * 1e3}
print(json.dumps(out, indent=1))
