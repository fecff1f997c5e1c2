"""Time one cfg5 leaf level (a level-1 node: 7 products of n/2, tf32 + 2 x bf16 RAW
leaves on CTA pairs, C-combination fused) with CUDA events; kernel-family split.
Usage: python tools/leaf_time.py [n=8192] [reps=20]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import strassen as S
from paper_2011_01441_b200.device import View

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
bt = b.t().contiguous()
c = torch.zeros(n, n, device="cuda")
st = torch.cuda.current_stream()


def run():
    S._leaf_level_b2raw(View.of(a), View.of(bt), [(View.of(c), 1)], st)


for _ in range(3):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
with nat.kernel_timing() as kt:
    run()
    torch.cuda.synchronize()
    tc = kt.read(nat.KT_TC_GEMM)
    lc = kt.read(nat.KT_LINCOMB)
h = n // 2
tf32eq = 7 * 2 * h * h * h * 2   # 2 tf32-equivalents per product (hi.hi tf32 + two bf16 corrections)
ts.sort()
med = ts[len(ts) // 2]
print(json.dumps({"n": n, "ms_median": med, "ms_min": ts[0], "leaf_kernel_ms": tc, "lincomb_ms": lc,
                  "tf32eq_tflops_kernel": tf32eq / (tc[0] * 1e-3) / 1e12 if tc[0] else None}))
