"""Fixed per-launch cost of the SIMT semiring kernel: CUDA-graph time of tiny
problems (one 128x128 tile, k = 4 .. 256) for the 32- and 64-bit kernels, and
of an empty-ish elementwise fill for comparison (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_fill, launch_mm


def graph_us(fn, reps=50):
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        with torch.cuda.graph(g, stream=s2):
            for _ in range(reps):
                fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


out = {}
for name, sr, dt, cdt in (("minplus32", nat.SR_MINPLUS_SAT32, torch.int32, torch.int32),
                          ("int_i32_i64", nat.SR_INT_I32_I64, torch.int32, torch.int64)):
    for n, k in ((128, 4), (128, 64), (128, 256), (384, 256)):
        a = torch.randint(0, 9, (n, k), device="cuda", dtype=dt)
        b = torch.randint(0, 9, (k, n), device="cuda", dtype=dt)
        c = torch.zeros(n, n, device="cuda", dtype=cdt)
        out[f"{name}_n{n}_k{k}"] = graph_us(
            lambda: launch_mm(sr, torch.cuda.current_stream(), View.of(a), View.of(b), View.of(c)))
c = torch.zeros(128, 128, device="cuda", dtype=torch.int32)
out["fill_128x128"] = graph_us(lambda: launch_fill(nat.SR_MINPLUS_SAT32, torch.cuda.current_stream(), View.of(c)))
print({k: round(v, 2) for k, v in out.items()})
