"""min-plus kernel time per C shape, alone and with a concurrent pinned H2D copy
(dev tool: explains the e2e pipeline's chunk costs).  Args: NxMxK ..."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

hsrc = torch.empty((8192, 8192), dtype=torch.int32).pin_memory()
hdst = torch.empty((8192, 8192), dtype=torch.int32, device="cuda")
side = torch.cuda.Stream()
for spec in sys.argv[1:] or ["8192x8192x8192", "8192x8192x256", "8192x8192x2048", "1024x8192x2048", "2048x4096x8192"]:
    n, m, k = (int(x) for x in spec.split("x"))
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randint(0, 2**20, (n, k), device="cuda", dtype=torch.int32, generator=g)
    B = torch.randint(0, 2**20, (k, m), device="cuda", dtype=torch.int32, generator=g)
    C = torch.full((n, m), 2**30, device="cuda", dtype=torch.int32)
    st = torch.cuda.current_stream()
    a, b, c = View.of(A), View.of(B), View.of(C)
    res = []
    for copy in ((False,) if os.environ.get("NOCOPY") else (False, True)):
        for _ in range(2):
            launch_mm(nat.SR_MINPLUS_SAT32, st, a, b, c)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            if copy:
                with torch.cuda.stream(side):
                    for _ in range(4):
                        hdst.copy_(hsrc, non_blocking=True)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); launch_mm(nat.SR_MINPLUS_SAT32, st, a, b, c); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
            torch.cuda.synchronize()
        res.append(min(ts))
    t = res[0]
    extra = f" | with H2D: {res[1]:.3f} ms ({res[1]/t:.2f}x)" if len(res) > 1 else ""
    print(f"{spec}: {t:.3f} ms {2*n*m*k/t/1e9:.1f} Top/s{extra}", flush=True)
