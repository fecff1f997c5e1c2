"""Minimal launcher for ncu captures: warm-up + a few paco_mm launches of one shape."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

sr = int(sys.argv[1]) if len(sys.argv) > 1 else nat.SR_MINPLUS_SAT32
n, m, k = (int(x) for x in (sys.argv[2:5] if len(sys.argv) > 4 else (8192, 8192, 8192)))
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
g = torch.Generator(device="cuda").manual_seed(0)
if sr in (nat.SR_MINPLUS_SAT32, nat.SR_MAXPLUS_SAT32):
    A = torch.randint(0, 2**20, (n, k), device="cuda", dtype=torch.int32, generator=g)
    B = torch.randint(0, 2**20, (k, m), device="cuda", dtype=torch.int32, generator=g)
    C = torch.full((n, m), 2**30, device="cuda", dtype=torch.int32)
elif sr == nat.SR_BF16_F32:
    A = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(k, m, device="cuda", generator=g).to(torch.bfloat16)
    C = torch.zeros(n, m, device="cuda", dtype=torch.float32)
else:
    A = torch.randn(n, k, device="cuda", generator=g)
    B = torch.randn(k, m, device="cuda", generator=g)
    C = torch.zeros(n, m, device="cuda")
st = torch.cuda.current_stream()
for _ in range(reps):
    launch_mm(sr, st, View.of(A), View.of(B), View.of(C), overwrite=(sr == nat.SR_BF16_F32))
torch.cuda.synchronize()
print("ok")
