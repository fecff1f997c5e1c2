"""Time the tcgen05 kernels (bf16 / 3xTF32) on a few shapes in a CUDA graph (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm


def graph_time(f, reps):
    st = torch.cuda.current_stream()
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            f()
    g.replay(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record(); g.replay(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best


for spec in sys.argv[1:] or ["bf16:65536x1024x256", "bf16:8192x8192x8192", "f32:4096x4096x4096"]:
    kind, dims = spec.split(":")
    n, m, k = (int(x) for x in dims.split("x"))
    dt = torch.bfloat16 if kind == "bf16" else torch.float32
    sr = nat.SR_BF16_F32 if kind == "bf16" else nat.SR_F32_TC
    a = torch.randn(n, k, device="cuda").to(dt); b = torch.randn(k, m, device="cuda").to(dt)
    c = torch.empty(n, m, device="cuda")
    av, bv, cv = View.of(a), View.of(b), View.of(c)
    reps = max(2, min(20, int(2e10 / (2 * n * m * k) + 1)))
    ms = graph_time(lambda: launch_mm(sr, torch.cuda.current_stream(), av, bv, cv, overwrite=True), reps)
    print(f"{spec}: {ms * 1e3:.1f} us  {2 * n * m * k / ms / 1e9:.1f} TFLOP/s", flush=True)
    del a, b, c
