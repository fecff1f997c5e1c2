"""§8f-f3: communication balance of GPU-level PACO plans, measured with ncu.

Runs every COMPUTE cuboid of mm_one_piece_partition(n, n, n, p) (and, for
comparison, a naive equal-rows split) as its own paco_mm launch on one GPU, in
a cudaProfilerStart/Stop range.  Under
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --csv
each launch's DRAM bytes are what that worker's GPU would move from HBM if it
ran the cuboid alone.  tools/comm_balance_report.py folds them into Q^max_p vs
Q^sum_p / p per plan (the paper's balance claim)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2011_01441_b200 import _native as nat
from paper_2011_01441_b200 import matmul as M
from paper_2011_01441_b200.device import View
from paper_2011_01441_b200.mm import launch_mm

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
ps = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,3,5,7,8").split(",")]
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randint(0, 2**20, (n, n), device="cuda", dtype=torch.int32, generator=g)
B = torch.randint(0, 2**20, (n, n), device="cuda", dtype=torch.int32, generator=g)
C = torch.full((n, n), 2**30, device="cuda", dtype=torch.int32)
a, b, c = View.of(A), View.of(B), View.of(C)
st = torch.cuda.current_stream()
layout = []
def cuboids(p, kind):
    if kind == "one_piece":
        plan = M.mm_one_piece_partition(n, n, n, p)
        return [(t.workers()[0], t.region) for t in plan.tasks if t.kind == "compute"]
    rows = [n * w // p for w in range(p + 1)]  # equal row slabs: the non-PACO baseline
    return [(w, M.Cuboid(rows[w], 0, 0, rows[w + 1] - rows[w], n, n)) for w in range(p)]
launch_mm(nat.SR_MINPLUS_SAT32, st, a.sub(0, 0, 256, 256), b.sub(0, 0, 256, 256), c.sub(0, 0, 256, 256))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for p in ps:
    for kind in ("one_piece", "row_slabs"):
        for w, cb in cuboids(p, kind):
            launch_mm(nat.SR_MINPLUS_SAT32, st, a.sub(cb.i0, cb.l0, cb.n, cb.k), b.sub(cb.l0, cb.j0, cb.k, cb.m),
                      c.sub(cb.i0, cb.j0, cb.n, cb.m), flags=nat.MM_ATOMIC if cb.l0 or cb.k < n else 0)
            layout.append({"p": p, "plan": kind, "worker": w, "n": cb.n, "m": cb.m, "k": cb.k})
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
json.dump({"n": n, "launches": layout}, open(os.environ.get("LAYOUT", "gpurun_out/comm_layout.json"), "w"))
print("ok", len(layout))
