"""Host<->device copy bandwidth from pinned memory, and the e2e pipeline's pieces."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
n = 8192
h = torch.empty((n, n), dtype=torch.int32).pin_memory()
d = torch.empty((n, n), dtype=torch.int32, device="cuda")
for name, f in [("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(3)]; e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name} 256 MiB: {ms:.2f} ms = {n*n*4/ms/1e6:.1f} GB/s", flush=True)
# concurrent H2D + D2H
h2 = torch.empty((n, n), dtype=torch.int32).pin_memory()
d2 = torch.empty((n, n), dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D || D2H 256 MiB each: {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
