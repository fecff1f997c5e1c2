"""Sweep the k-phased host pipeline's shape (PACO_PIPE_KP) on cfg2's e2e call.

For each "first,growth,cap,share,R" setting, times `mm_seq` on pinned host
operands (n=m=k=8192, (min,+)) exactly as bench.py's e2e leg does, and prints
the median ms; also prints the device time of the chunk kernels so the
host-side cost model can be calibrated.

    python tools/kp_sweep.py "128,2,2048,0.25,16" "128,3,3072,0.375,8" ...
"""

import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200 import mm as MM
from paper_2011_01441_b200.device import View


def main():
    n = 8192
    rng = np.random.default_rng(1002)
    A = rng.integers(0, 2**20, (n, n), dtype=np.int32)
    B = rng.integers(0, 2**20, (n, n), dtype=np.int32)
    Ah = torch.from_numpy(A).pin_memory()
    Bh = torch.from_numpy(B).pin_memory()
    C0 = torch.full((n, n), 2**30, dtype=torch.int32).pin_memory()
    Ch = torch.empty_like(C0).pin_memory()
    st = torch.cuda.current_stream()

    # chunk kernel device times (whole C, k = w) and tail blocks (rows r, k = w)
    a = Ah.cuda()
    b = Bh.cuda()
    c = C0.cuda()
    av, bv, cv = View.of(a), View.of(b), View.of(c)
    for rows, w in [(n, 128), (n, 256), (n, 384), (n, 512), (n, 1024), (n, 2048), (n, 3072), (n, 8192),
                    (512, 2048), (1024, 1024), (1024, 2048), (1024, 3072), (768, 2048), (2048, 2048)]:
        fn = lambda: MM.launch_mm(nat.SR_MINPLUS_SAT32, st, av.sub(0, 0, rows, w), bv.sub(0, 0, w, n),
                                  cv.sub(0, 0, rows, n))
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        ideal = 31.56 * rows * w / n / n
        print(f"kernel rows={rows} k={w}: {ms:.3f} ms (pro-rata of 31.56: {ideal:.3f}, eff {ideal / ms:.3f})",
              flush=True)
    del a, b, c
    torch.cuda.synchronize()

    for kp in sys.argv[1:] or ["128,2,2048,0.25,16"]:
        MM._KP = tuple(float(x) for x in kp.split(","))
        ts = []
        for it in range(4):
            Ch.copy_(C0)
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            M.mm_seq(Ah, Bh, Ch, M.SEMIRING_MINPLUS_SAT)
            f1.record()
            f1.synchronize()
            if it:
                ts.append(f0.elapsed_time(f1))
        print(f"KP={kp}: e2e median {statistics.median(ts):.3f} ms  ({[round(t, 2) for t in ts]})", flush=True)


if __name__ == "__main__":
    main()
