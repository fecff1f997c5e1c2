"""cfg2 end to end (NumPy mm_seq) with uniform vs geometric last-phase row blocks (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2011_01441_b200 import mm as M

for decay, front in ((None, None), (0.7, None), (0.6, None), (None, None), (0.7, None)):
    M._ROW_DECAY = decay
    r = bench.e2e_numpy_cfg2(0, 5)
    print("decay", decay, "ms", round(r["ms_per_step"], 3), [round(x, 2) for x in r["ms_all"]], flush=True)
