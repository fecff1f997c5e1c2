"""Back-to-back tcgen05 bf16 launches (cfg3 shape) traced into separate buffers
(paco_debug_trace stamps): how far the second launch's start overlaps the
first launch's drain (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

n, m, k = 65536, 1024, 256
a = torch.randn(n, k, device="cuda").to(torch.bfloat16)
b = torch.randn(k, m, device="cuda").to(torch.bfloat16)
c = torch.empty(n, m, device="cuda")
st = torch.cuda.current_stream()
lib = nat.load()
for _ in range(5):
    launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c), overwrite=True)
L = 3
trs = [torch.zeros(148 * 16 * 6, dtype=torch.int64, device="cuda") for _ in range(L)]
torch.cuda.synchronize()
for tr in trs:
    nat.check(lib.paco_debug_trace(tr.data_ptr()))
    launch_mm(nat.SR_BF16_F32, st, View.of(a), View.of(b), View.of(c), overwrite=True)
nat.check(lib.paco_debug_trace(None))
torch.cuda.synchronize()
ts = [tr.view(148, 16, 6).cpu().numpy().astype(np.float64) for tr in trs]
t0 = min(t[t > 0].min() for t in ts)
for j, t in enumerate(ts):
    t = np.where(t > 0, (t - t0) / 1e3, np.nan)
    life = t[:, 15]
    tiles = t[:, :15]
    e0 = tiles[:, 0, 4]  # first accumulator ready
    e1_first = tiles[:, 0, 5]
    last_e1 = np.nanmax(tiles[:, :, 5], axis=1)
    print(f"launch {j}: entry min {np.nanmin(life[:, 0]):.2f} med {np.nanmedian(life[:, 0]):.2f} max {np.nanmax(life[:, 0]):.2f}"
          f" | wait done (setup) med {np.nanmedian(life[:, 1]):.2f} max {np.nanmax(life[:, 1]):.2f}"
          f" | first acc ready med {np.nanmedian(e0):.2f} | first tile stores issued min {np.nanmin(e1_first):.2f}"
          f" med {np.nanmedian(e1_first):.2f}"
          f" | last stores issued min {np.nanmin(last_e1):.2f} med {np.nanmedian(last_e1):.2f} max {np.nanmax(last_e1):.2f}"
          f" | exit min {np.nanmin(life[:, 2]):.2f} med {np.nanmedian(life[:, 2]):.2f} max {np.nanmax(life[:, 2]):.2f}")
    print("   producer: first claim med %.2f, B issued med %.2f | tile0: P0 first A load %.2f, P1 last A load %.2f, "
          "M0 stage ready %.2f, M1 mma issued %.2f, E0 acc ready %.2f, E1 stores issued %.2f (medians)"
          % tuple([np.nanmedian(life[:, 3]), np.nanmedian(life[:, 4])] + [np.nanmedian(tiles[:, 0, f]) for f in range(6)]))
    print("   tile1: " + " ".join("%.2f" % np.nanmedian(tiles[:, 1, f]) for f in range(6)))
    ntiles = np.sum(~np.isnan(tiles[:, :, 4]), axis=1)
    print("   tiles per CTA (first 15 traced):", np.bincount(ntiles))
