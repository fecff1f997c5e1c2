"""Per-tile timeline of the tcgen05 bf16 kernel (paco_debug_trace stamps):
producer first/last load issue, MMA first stage ready / last MMA issued,
epilogue accumulator ready / last store issued (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

n, m, k = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (65536, 1024, 256)))
a = torch.randn(n, k, device="cuda").to(torch.bfloat16)
b = torch.randn(k, m, device="cuda").to(torch.bfloat16)
c = torch.empty(n, m, device="cuda")
st = torch.cuda.current_stream()
for _ in range(3):
    launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c), overwrite=True)
tr = torch.zeros(148 * 16 * 6, dtype=torch.int64, device="cuda")
lib = nat.load()
nat.check(lib.paco_debug_trace(tr.data_ptr()))
launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c), overwrite=True)
torch.cuda.synchronize()
nat.check(lib.paco_debug_trace(None))
t = tr.view(148, 16, 6).cpu().numpy().astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1e3, np.nan)   # us
life = t[:, 15, :6]
print("producer: first claim done median %.2f, resident B issued median %.2f us"
      % (np.nanmedian(life[:, 3]), np.nanmedian(life[:, 4])))
t = t[:, :15]
print("CTA entry: min %.2f max %.2f | setup done: median %.2f | exit: min %.2f median %.2f max %.2f us"
      % (np.nanmin(life[:, 0]), np.nanmax(life[:, 0]), np.nanmedian(life[:, 1]), np.nanmin(life[:, 2]),
         np.nanmedian(life[:, 2]), np.nanmax(life[:, 2])))
print("fields: P0 first-load  P1 last-load  M0 stage-ready  M1 mma-issued  E0 acc-ready  E1 stores-issued (us)")
for cta in (0, 1, 74, 147):
    print(f"CTA {cta}")
    for i in range(15):
        if np.isnan(t[cta, i]).all():
            continue
        print("  tile %2d " % i + " ".join("%7.2f" % x for x in t[cta, i]))
e1 = np.nanmax(t[:, :, 5], axis=1)
print("kernel end (last E1) per CTA: min %.2f median %.2f max %.2f us" % (np.nanmin(e1), np.nanmedian(e1), np.nanmax(e1)))
d = t[:, 1:, 4] - t[:, :-1, 4]
print("median tile period (E0 spacing) %.2f us; median epilogue E1-E0 %.2f us; median MMA M1-M0 %.2f us; median load->ready M0-P0 %.2f us"
      % (np.nanmedian(d), np.nanmedian(t[:, :, 5] - t[:, :, 4]), np.nanmedian(t[:, :, 3] - t[:, :, 2]), np.nanmedian(t[:, :, 2] - t[:, :, 0])))
