"""Dev timing: cuBLAS bf16->bf16 and bf16->f32 (out_dtype) on the cfg3 shape, and a 256 MB fill, in CUDA graphs."""
import torch
n, m, k = 65536, 1024, 256
a = torch.randn(n, k, device="cuda").to(torch.bfloat16)
b = torch.randn(k, m, device="cuda").to(torch.bfloat16)
def t(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps): f()
    g.replay(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); g.replay(); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    return best
c16 = torch.empty(n, m, device="cuda", dtype=torch.bfloat16)
print("cublas bf16->bf16: %.1f us" % t(lambda: torch.mm(a, b, out=c16)))
try:
    c32 = torch.empty(n, m, device="cuda", dtype=torch.float32)
    print("cublas bf16->f32 (out_dtype): %.1f us" % t(lambda: torch.mm(a, b, out_dtype=torch.float32)))
except Exception as e:
    print("out_dtype unsupported:", e)
af, bf = a.float(), b.float()
c = torch.empty(n, m, device="cuda")
print("fill f32 256MB: %.1f us" % t(lambda: c.fill_(1.0)))
