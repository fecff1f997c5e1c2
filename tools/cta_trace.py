"""Per-CTA timing of one paco_mm launch (smid, duration, stage count) -> balance report."""
import sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

sr = int(sys.argv[1]); n, m, k = (int(x) for x in sys.argv[2:5])
g = torch.Generator(device="cuda").manual_seed(0)
if sr == nat.SR_F32:
    A = torch.randn(n, k, device="cuda", generator=g); B = torch.randn(k, m, device="cuda", generator=g)
    C = torch.zeros(n, m, device="cuda")
else:
    A = torch.randint(0, 2**20, (n, k), device="cuda", dtype=torch.int32, generator=g)
    B = torch.randint(0, 2**20, (k, m), device="cuda", dtype=torch.int32, generator=g)
    C = torch.full((n, m), 2**30, device="cuda", dtype=torch.int32)
tr = torch.zeros(10 * 8192, dtype=torch.int64, device="cuda")
lib = nat.load()
st = torch.cuda.current_stream()
launch_mm(sr, st, View.of(A), View.of(B), View.of(C))
nat.check(lib.paco_debug_trace(tr.data_ptr()))
launch_mm(sr, st, View.of(A), View.of(B), View.of(C))
torch.cuda.synchronize()
nat.check(lib.paco_debug_trace(None))
t = tr.view(-1, 10).cpu().numpy()
t = t[t[:, 2] > 0]
host = nat.plan_cta(sr, n, m, k, len(t))
print("device pieces == host paco_plan_cta:", [tuple(r) for r in t[:, 4:10]] == [tuple(h) for h in host])
t0 = t[:, 1].min()
dur = (t[:, 2] - t[:, 1]) / 1e6
print(f"ctas={len(t)} span={(t[:,2].max()-t0)/1e6:.2f} ms  dur min/mean/max = {dur.min():.2f}/{dur.mean():.2f}/{dur.max():.2f} ms")
print("start offsets (ms) max:", (t[:, 1].max() - t0) / 1e6)
per_sm = collections.defaultdict(list)
for i, row in enumerate(t):
    per_sm[int(row[0])].append(i)
print("SMs used:", len(per_sm), "ctas/SM histogram:", collections.Counter(len(v) for v in per_sm.values()))
work = t[:, 3]
print("stages/CTA min/mean/max:", work.min(), work.mean(), work.max())
rate = work / dur
print("stages per ms min/mean/max: %.1f %.1f %.1f" % (rate.min(), rate.mean(), rate.max()))
slow = np.argsort(-dur)[:8]
for i in slow:
    sm = int(t[i, 0]); mates = [j for j in per_sm[sm] if j != i]
    print(f"cta {i} sm {sm} dur {dur[i]:.2f} stages {work[i]} start {(t[i,1]-t0)/1e6:.2f}  mate(s) {[(j, round(dur[j],2), int(work[j])) for j in mates]}")
fast = np.argsort(dur)[:4]
for i in fast:
    sm = int(t[i, 0]); mates = [j for j in per_sm[sm] if j != i]
    print(f"FAST cta {i} sm {sm} dur {dur[i]:.2f} stages {work[i]}  mate(s) {[(j, round(dur[j],2), int(work[j])) for j in mates]}")
