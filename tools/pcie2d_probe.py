"""H2D throughput of 2-D (strided) copies from pinned memory vs row width."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_01441_b200.mm import _copy2d
n = 8192
h = torch.empty((n, n), dtype=torch.int32).pin_memory()
d = torch.empty((n, n), dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
for w in (256, 512, 1024, 2048, 4096, 8192):
    f = lambda: _copy2d(st, d, 0, 0, h, 0, 0, n, w)
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(3)]; e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"H2D {n}x{w} int32 (row {w*4} B): {ms:.3f} ms = {n*w*4/ms/1e6:.1f} GB/s", flush=True)
