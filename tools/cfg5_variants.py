"""cfg5 (Strassen fp32 n=16384, 2 levels) per leaf format: bf16x3 on pre-split
planes (default) vs tf32 + 2 x bf16 on raw fp32 operands -- step time,
per-kernel-family time, error on sampled rows vs f64."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import strassen as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
g = torch.Generator(device="cuda").manual_seed(1005)
a = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
b = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
rows = torch.arange(0, n, n // 64, device="cuda")
ref = a[rows].double() @ b.double()
res = {}
for name, b3, direct in (("bf16x3_direct", True, True), ("bf16x3_level1", True, False), ("tf32b2_raw", False, False),
                         ("bf16x3_direct_again", True, True)):
    S.LEAF_BF16X3, S.B3_DIRECT = b3, direct
    for _ in range(2):
        c = S.strassen_seq(a, b, n, base=n // 4)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = S.strassen_seq(a, b, n, base=n // 4)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    with nat.kernel_timing() as kt:
        S.strassen_seq(a, b, n, base=n // 4)
        torch.cuda.synchronize()
        fam = {f: kt.read(i) for f, i in (("tc", 1), ("split", 2), ("lincomb", 3), ("elementwise", 4))}
    res[name] = {"ms": sorted(ts), "kernels_ms": {k: round(v[0], 3) for k, v in fam.items()},
                 "rel_err_rows": float((c[rows].double() - ref).norm() / ref.norm())}
    print(name, json.dumps(res[name]), flush=True)
print(json.dumps(res))
