"""Time paco_mm for several CTA-level plan sizes p (pieces from paco_plan_cta)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

sr = int(sys.argv[1]); n, m, k = (int(x) for x in sys.argv[2:5]); ps = [int(x) for x in sys.argv[5].split(",")]
g = torch.Generator(device="cuda").manual_seed(0)
if sr == nat.SR_F32:
    A = torch.randn(n, k, device="cuda", generator=g); B = torch.randn(k, m, device="cuda", generator=g)
    C = torch.zeros(n, m, device="cuda")
else:
    A = torch.randint(0, 2**20, (n, k), device="cuda", dtype=torch.int32, generator=g)
    B = torch.randint(0, 2**20, (k, m), device="cuda", dtype=torch.int32, generator=g)
    C = torch.full((n, m), 2**30, device="cuda", dtype=torch.int32)
st = torch.cuda.current_stream()
a, b, c = View.of(A), View.of(B), View.of(C)
for p in ps:
    pieces = nat.plan_cta(sr, n, m, k, p)
    for _ in range(2):
        launch_mm(sr, st, a, b, c, pieces=pieces)
    ts = []
    for _ in range(4):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); launch_mm(sr, st, a, b, c, pieces=pieces); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts)
    print(f"sr={sr} {n}x{m}x{k} p={p}: {t:.3f} ms  {2*n*m*k/t/1e9:.1f} Top/s", flush=True)
