"""cfg3 bf16 kernel: back-to-back launches vs a CUDA graph of the same launches
(host launch gap), and host time per paco_mm call (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

n, m, k = 65536, 1024, 256
a = torch.randn(n, k, device="cuda").to(torch.bfloat16)
b = torch.randn(k, m, device="cuda").to(torch.bfloat16)
c = torch.empty(n, m, device="cuda")
av, bv, cv = View.of(a), View.of(b), View.of(c)
st = torch.cuda.Stream()
reps = 20
with torch.cuda.stream(st):
    for _ in range(3):
        launch_mm(nat.SR_BF16_F32, st, av, bv, cv, overwrite=True)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(reps):
        launch_mm(nat.SR_BF16_F32, st, av, bv, cv, overwrite=True)
    e1.record(st)
    host = (time.perf_counter() - t0) / reps * 1e6
    e1.synchronize()
    print(f"direct: {e0.elapsed_time(e1) / reps * 1e3:.1f} us/launch on device, host {host:.1f} us/call")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            launch_mm(nat.SR_BF16_F32, st, av, bv, cv, overwrite=True)
    g.replay(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0.record(st); g.replay(); e1.record(st); e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    print(f"graph:  {best:.1f} us/launch")
