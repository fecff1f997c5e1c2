"""One paco_strassen_split49 pass at cfg5's size (A side, 16384^2 operand) for ncu (dev tool)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2011_01441_b200 import _native as nat

n, h = 16384, 4096
x = torch.rand(n, n, device="cuda") * 2 - 1
planes = torch.empty((2, 49, h, h), dtype=torch.bfloat16, device="cuda")
his = (ctypes.c_void_p * 49)(*[planes[0, o].data_ptr() for o in range(49)])
los = (ctypes.c_void_p * 49)(*[planes[1, o].data_ptr() for o in range(49)])
st = torch.cuda.current_stream().cuda_stream
for side in (0, 1, 0):
    nat.check(nat.load().paco_strassen_split49(0, st, side, x.data_ptr(), n, h, his, los, h))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    nat.check(nat.load().paco_strassen_split49(0, st, 0, x.data_ptr(), n, h, his, los, h))
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 5
byts = n * n * 4 + 49 * h * h * 4
print(f"split49: {ms:.3f} ms, {byts / ms / 1e6:.0f} GB/s (1 GiB read + 49 x 2 bf16 planes written)")
