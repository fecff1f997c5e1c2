"""Tropical 8192^3 (cfg2) and 16384^3 (cfg4) device time of the SIMT kernel --
run twice with PACO_DEV_KNOBS=1 PACO_SIMT_TMA=0/1 for the TMA-ring A/B."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

res = {}
for name, kid, n, reps in (("cfg2", nat.SR_MINPLUS_SAT32, 8192, 10), ("cfg4", nat.SR_MAXPLUS_SAT32, 16384, 2)):
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randint(0, 1 << 20, (n, n), device="cuda", dtype=torch.int32, generator=g)
    b = torch.randint(0, 1 << 20, (n, n), device="cuda", dtype=torch.int32, generator=g)
    c = torch.empty(n, n, device="cuda", dtype=torch.int32)
    st = torch.cuda.current_stream()
    f = lambda: launch_mm(kid, st, View.of(a), View.of(b), View.of(c), overwrite=True)  # noqa: E731
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[name] = {"ms": ms, "top_s": 2 * n ** 3 / ms / 1e9, "checksum": int(c.long().sum().item())}
    del a, b, c
print(json.dumps({"tma": os.environ.get("PACO_SIMT_TMA", "default"), **res}))
