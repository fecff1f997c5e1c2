"""cfg5 step time: fused-producer leaves vs the split path (same process)."""
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
res = {}
for fused in (True, False, True):
    S.FUSED_PRODUCER = fused
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
    rows = torch.arange(0, n, n // 64, device="cuda")
    ref = a[rows].double() @ b.double()
    err = float((c[rows].double() - ref).norm() / ref.norm())
    res[f"fused={fused}"] = {"ms": sorted(ts), "kernels": fam, "rel_err_rows": err}
print(json.dumps(res, indent=1))
