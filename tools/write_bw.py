"""Write bandwidth of a plain fill and a copy (the HBM write ceiling the cfg3 epilogue is compared with)."""
import torch
for mb in (268, 1073):
    n = mb * 1024 * 1024 // 4
    c = torch.empty(n, device="cuda")
    for _ in range(3): c.fill_(1.0)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): c.fill_(2.0)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"fill {mb} MiB: {ms*1e3:.1f} us  {n*4/ms/1e6:.0f} GB/s")
    a = torch.empty(n // 2, device="cuda"); b = torch.empty(n // 2, device="cuda")
    for _ in range(3): b.copy_(a)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): b.copy_(a)
    e1.record(); e1.synchronize(); ms = e0.elapsed_time(e1) / 20
    print(f"copy {mb//2} MiB: {ms*1e3:.1f} us  {n*4/ms/1e6:.0f} GB/s (r+w)")
