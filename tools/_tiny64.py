import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm
n, k = 128, 4
a = torch.randint(0, 9, (n, k), device="cuda", dtype=torch.int32)
b = torch.randint(0, 9, (k, n), device="cuda", dtype=torch.int32)
c = torch.zeros(n, n, device="cuda", dtype=torch.int64)
for _ in range(3):
    launch_mm(nat.SR_INT_I32_I64, torch.cuda.current_stream(), View.of(a), View.of(b), View.of(c))
torch.cuda.synchronize()
