"""cfg5 step: host enqueue time vs device time, and the device timeline's idle
gaps between kernels (torch.profiler / CUPTI kernel and memset records)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2011_01441_b200 import strassen as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
a = torch.rand(n, n, device="cuda") * 2 - 1
b = torch.rand(n, n, device="cuda") * 2 - 1
for _ in range(3):
    S.strassen_seq(a, b, n, base=n // 4)
torch.cuda.synchronize()
host, dev = [], []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    t0 = time.perf_counter()
    S.strassen_seq(a, b, n, base=n // 4)
    host.append((time.perf_counter() - t0) * 1e3)
    e1.record()
    e1.synchronize()
    dev.append(e0.elapsed_time(e1))
print(json.dumps({"host_enqueue_ms": host, "device_ms": dev}))

from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        S.strassen_seq(a, b, n, base=n // 4)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
rows = []
prev_end = None
for e in evs:
    st, en = e.time_range.start, e.time_range.end
    gap = None if prev_end is None else st - prev_end
    rows.append((round(st / 1e3, 3), round((en - st) / 1e3, 3), None if gap is None else round(gap / 1e3, 3),
                 e.name[:60]))
    prev_end = en if prev_end is None else max(prev_end, en)
half = len(rows) // 2
tot_gap = sum(r[2] for r in rows[half + 1:] if r[2] and r[2] > 0)
print(json.dumps({"events": len(rows), "second_step_gap_ms": tot_gap}))
for r in rows[half:]:
    print(r)
