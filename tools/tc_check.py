"""Dev check of the tcgen05 bf16 kernel: relative error vs float64 product, and timing."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

torch.manual_seed(0)
for (n, m, k, ow) in [(128, 256, 64, True), (256, 192, 128, True), (300, 500, 200, True), (300, 500, 200, False),
                      (1000, 1024, 256, True), (65536, 1024, 256, True)]:
    a = torch.randn(n, k, device="cuda").to(torch.bfloat16)
    b = torch.randn(k, m, device="cuda").to(torch.bfloat16)
    c0 = torch.randn(n, m, device="cuda") if not ow else torch.zeros(n, m, device="cuda")
    c = c0.clone()
    M.mm_seq(a, b, c, M.SEMIRING_BF16, overwrite=ow)
    torch.cuda.synchronize()
    ref = a.double() @ b.double() + c0.double()
    err = ((c.double() - ref).norm() / ref.norm()).item()
    print(f"{n}x{m}x{k} overwrite={ow}: rel err {err:.3e}", flush=True)
n, m, k = 65536, 1024, 256
a = torch.randn(n, k, device="cuda").to(torch.bfloat16); b = torch.randn(k, m, device="cuda").to(torch.bfloat16)
c = torch.zeros(n, m, device="cuda")
st = torch.cuda.current_stream()
for _ in range(3):
    launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c), overwrite=True)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c), overwrite=True); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
t = min(ts)
byt = 2 * n * k + 2 * k * m + 4 * n * m
print(f"cfg3 {n}x{m}x{k}: {t*1e3:.1f} us  {2*n*m*k/t/1e9:.1f} TFLOP/s  {byt/t/1e6:.0f} GB/s (alg bytes)")
