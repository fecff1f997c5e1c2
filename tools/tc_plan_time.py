"""mm_execute of GPU-level plans with the tcgen05 kinds on ONE device: concurrent
persistent launches on the plan's worker streams vs one launch (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_01441_b200 import matmul as M

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
for name, sem, dt in (("f32 3xTF32", M.SEMIRING_F32, torch.float32), ("bf16", M.SEMIRING_BF16, torch.bfloat16)):
    a = torch.randn(n, n, device="cuda").to(dt); b = torch.randn(n, n, device="cuda").to(dt)
    c = torch.zeros(n, n, device="cuda")
    for p in (1, 3, 5, 8):
        plan = M.mm_one_piece_partition(n, n, n, p)
        for mode in ("serial_sim", "parallel"):
            M.mm_execute(plan, a, b, c, sem, mode=mode); torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(3):
                M.mm_execute(plan, a, b, c, sem, mode=mode)
            torch.cuda.synchronize()
            print(f"{name} p={p} {mode}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms", flush=True)
