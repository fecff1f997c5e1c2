"""NumPy e2e of cfg2 (bench.e2e_numpy_cfg2) in a fresh process vs after the bench's
device work, and vs staging thread counts."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2011_01441_b200 import mm as MM

res = {"host_threads": MM._HOST_THREADS, "torch_threads": torch.get_num_threads()}
res["fresh"] = bench.e2e_numpy_cfg2(0, 5)["ms_all"]
x = torch.randint(0, 2**20, (8192, 8192), dtype=torch.int32, device="cuda")
xh = x.cpu().pin_memory()
res["after_pin_copy"] = bench.e2e_numpy_cfg2(0, 5)["ms_all"]
for t in (10, 14, 16):
    MM._HOST_THREADS = t
    res[f"threads_{t}"] = bench.e2e_numpy_cfg2(0, 3)["ms_all"]
print(json.dumps(res))
