"""cfg3 bf16 launch: eager back-to-back vs the same launches replayed from a
CUDA graph (separates host launch cost from GPU time) (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

n, k, m = 65536, 256, 1024
a = torch.randn(n, k, device="cuda").to(torch.bfloat16)
b = torch.randn(k, m, device="cuda").to(torch.bfloat16)
c = torch.empty(n, m, device="cuda")
st = torch.cuda.Stream()
R = 20
with torch.cuda.stream(st):
    fn = lambda: launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c), overwrite=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(R):
        fn()
    e1.record(st)
    e1.synchronize()
    eager = e0.elapsed_time(e1) / R * 1e3
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(R):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0.record(st)
    g.replay()
    e1.record(st)
    e1.synchronize()
    graph = e0.elapsed_time(e1) / R * 1e3
print({"eager_us": eager, "graph_us": graph})
