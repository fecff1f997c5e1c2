"""(+,x) f64 / int64 / f32-SIMT kernel rates at 4096^3 (dev tool: the non-config semirings)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
for name, sr, dt in (("f64", nat.SR_F64, torch.float64), ("int64", nat.SR_INT_I64, torch.int64),
                     ("f32_simt", nat.SR_F32, torch.float32), ("int32->64", nat.SR_INT_I32_I64, torch.int32),
                     ("minplus_i64", nat.SR_MINPLUS_I64, torch.int64)):
    if dt.is_floating_point:
        a = torch.randn(n, n, device="cuda", dtype=dt); b = torch.randn(n, n, device="cuda", dtype=dt)
    else:
        a = torch.randint(-100, 100, (n, n), device="cuda", dtype=dt); b = torch.randint(-100, 100, (n, n), device="cuda", dtype=dt)
    cdt = torch.int64 if dt == torch.int32 else dt
    c = torch.zeros(n, n, device="cuda", dtype=cdt)
    st = torch.cuda.current_stream()
    f = lambda: launch_mm(sr, st, View.of(a), View.of(b), View.of(c))
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); f(); f(); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 2
    print(f"{name}: {ms:.2f} ms  {2 * n**3 / ms / 1e9:.1f} T(fl)op/s", flush=True)
if dt is not None:
    a = torch.randn(n, n, device="cuda", dtype=torch.float64); b = torch.randn(n, n, device="cuda", dtype=torch.float64)
    torch.mm(a, b); torch.cuda.synchronize()
    e0.record(); torch.mm(a, b); torch.mm(a, b); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 2
    print(f"cuBLAS f64 dgemm: {ms:.2f} ms  {2 * n**3 / ms / 1e9:.1f} TFLOP/s")
